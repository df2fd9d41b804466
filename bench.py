#!/usr/bin/env python
"""Benchmark of the B200 MISDC / PMISDC sweep engine (driver contract: one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c5] [--scale 1]

Workload (``config.workload``): BASELINE.json config 5 by default -- 3-D periodic 256^3 x 9 species
mass-action ADR, 7 Gauss-Lobatto nodes (M = 6), 10 sweeps per step, PMISDC = CISDCQ nu = 1 with the
D(m+1) || R(m) streams, multigrid to 1e-10 -- the largest configuration, on which BASELINE.md
places the roofline claims (configs 1-2 are L2-resident / launch-bound; they are parity cases).
A bench "step" is one SDC time step (initialise from phi^0, 10 sweeps): every step does identical
work.  Metric: cell-species-node updates per second per sweep = n * M * sweeps / time.

  value     device-resident inputs (cisdc_gpu_integrate_device), CUDA-event time on the engine's
            stream, max over ranks; fields are >> L2 (1.2 GB each), no flush needed.
  e2e       the reference-facing C-ABI call with HOST pinned buffers (cisdc_gpu_integrate): the
            H2D of phi^0 and the D2H of the final state are inside every timed step.
  roofline  dominant kernel class by live CUDA-event time; achieved = algorithmic bytes (HBM) or
            analytic FP64 flops (Newton/LU) per launch / average launch time.
  cpu_baseline  the UNMODIFIED reference (oracle/_ref, built from /root/reference) on a bounded
            sample of the same workload (scaled grid), 1 core, rank 0 at N = 1.

Multi-GPU: replicas only (no data-path collective); value = sum over ranks.
--impl reference times the reference's CPU path (execute_pipelined with all useful host threads)
on a bounded sample per step.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# bounded CPU samples (grid scale divisor, steps) per config: ~10-30 s of reference CPU work
CPU_SAMPLE = {"c0": (1, 20), "c1": (1, 100), "c2": (4, 4), "c3": (8, 1), "c4": (16, 1), "c5": (8, 1)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--scheme", type=int, default=None, help="override the config's scheme")
    ap.add_argument("--workers", type=int, default=2, help="CISDCQ: >0 concurrent D/R streams")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(ws, v: float) -> float:
    if ws <= 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_reference_sample(cfg_name: str, scheme: int, workers: int, steps: int | None = None):
    """Run the reference CPU path on the bounded sample; returns (updates/s, seconds, sample text, kind, cores)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # test infrastructure: the reference / its port, only as the CPU baseline
    from paper_1801_01201_b200 import api, problems
    scale, nsteps = CPU_SAMPLE.get(cfg_name, (8, 1))
    if steps is not None:
        nsteps = steps
    spec = problems.CONFIGS[cfg_name](scale=scale) if cfg_name != "c0" else problems.config_c0()
    opt = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=nsteps, M=spec.M, n_sweeps=spec.n_sweeps,
                               nu=spec.nu, workers=workers)
    have_ref = oracle.ref_lib() is not None
    t0 = time.perf_counter()
    if have_ref:
        oracle.ref_integrate(spec.problem, spec.phi0, opt)
    else:
        oracle.integrate(spec.problem, spec.phi0, opt)
    dt = time.perf_counter() - t0
    updates = spec.problem.dim * spec.M * spec.n_sweeps * nsteps
    grid = "x".join(str(x) for x in spec.problem.n[: spec.problem.ndim])
    sample = (f"{cfg_name} scaled 1/{scale} per axis: {grid} cells x {spec.problem.nspecies} species, "
              f"{nsteps} step(s) x {spec.n_sweeps} sweeps, scheme {scheme}, workers {workers}")
    return updates / dt, dt, sample, "reference" if have_ref else "port", max(1, workers if workers > 0 else 1)


def workload_config(cfg_name: str, spec, scheme: int, workers: int) -> dict:
    """The bench line's config object: the grid that actually ran."""
    desc = spec.problem
    n = list(desc.n[: desc.ndim])
    dofs = int(np.prod(n)) * desc.nspecies
    return {"workload": f"{cfg_name}: {desc.name} {'x'.join(map(str, n))} x {desc.nspecies} species",
            "scheme": ["misdc", "misdcq", "cisdcq", "imexq"][scheme], "nu": spec.nu, "workers": workers, "M": spec.M,
            "sweeps_per_step": spec.n_sweeps, "dt": spec.dt, "dofs": dofs, "updates_per_step": dofs * spec.M * spec.n_sweeps,
            "l2": ("inputs larger than L2 (each field %.2f GB)" if 8 * dofs > 126e6 else
                   "fields fit in L2 (each field %.4f GB; no flush: the configuration itself is that small)")
            % (8 * dofs / 1e9)}


def run_reference_arm(args, ws, rank):
    """The reference's CPU path (oracle/_ref: unmodified cisdc::execute_pipelined / cisdc::integrate
    driving the oracle problem class) on a bounded sample of the workload, per step.  The line's
    config states what actually ran: the sampled grid, the thread count and the host's nproc."""
    if rank != 0:
        return
    from paper_1801_01201_b200 import problems
    sample_scale = CPU_SAMPLE.get(args.config, (8, 1))[0] if args.config != "c0" else 1
    spec = problems.CONFIGS[args.config](scale=sample_scale) if args.config != "c0" else problems.config_c0()
    scheme = spec.scheme if args.scheme is None else args.scheme
    nproc = os.cpu_count() or 1
    workers = min(nproc, max(2 * spec.nu, spec.M)) if scheme == 2 else 0
    for _ in range(args.warmup):
        cpu_reference_sample(args.config, scheme, workers, steps=1)
    times, rates = [], []
    sample = kind = None
    cores = 1
    for _ in range(args.steps):
        r, t, sample, kind, cores = cpu_reference_sample(args.config, scheme, workers, steps=1)
        times.append(t)
        rates.append(r)
    tot = float(np.sum(times))
    value = float(np.mean(rates))
    desc = spec.problem
    full_grid = "x".join(str(x * sample_scale) for x in desc.n[: desc.ndim])
    cfg = workload_config(args.config, spec, scheme, workers)
    cfg.update(parallelism=f"host threads x{cores}", nproc=nproc,
               sample_of=f"{args.config}: {desc.name} {full_grid} x {desc.nspecies} species",
               sample_scale_per_axis=f"1/{sample_scale}",
               note="the reference's CPU path on a bounded sample (scaled grid, 1 step per bench step); "
                    "the per-update rate is compared, not the wall time of the full workload")
    line = {
        "impl": "reference", "metric": "cell-species-node updates/s per SDC sweep (FP64)", "value": value,
        "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded BASELINE config generator)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": cores, "kind": kind, "sample": sample,
                         "nproc": nproc},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
        return
    import torch

    from paper_1801_01201_b200 import _abi, api, problems, roofline
    lib = _abi.load(build_if_missing=True)
    torch.cuda.set_device(local)
    spec = problems.CONFIGS[args.config](scale=args.scale) if args.config != "c0" else problems.config_c0()
    scheme = spec.scheme if args.scheme is None else args.scheme
    workers = args.workers if scheme == 2 else 0
    desc = spec.problem
    if scheme == 3:  # IMEXQ: the periodic ADR class's coupled stage (cisdc_gpu.h), the paper's baseline scheme
        import dataclasses
        desc = dataclasses.replace(desc, coupled_tol=1e-13, coupled_max_iter=60)
    n = desc.dim
    ctx = api.GpuContext(desc, spec.M, spec.convention)
    opt = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=spec.n_sweeps, nu=spec.nu,
                               workers=workers, convention=spec.convention)
    oc = opt.to_c()
    rep = _abi.StepReportC()
    incs = np.zeros(spec.n_sweeps)
    d_phi0 = torch.from_numpy(spec.phi0).to(f"cuda:{local}")
    d_out = torch.empty_like(d_phi0)
    torch.cuda.synchronize()

    # the per-kernel breakdown pass runs the sweeps serially on one stream (workers = 0) so that the event
    # intervals of different kernel classes never overlap
    oc1 = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=spec.n_sweeps, nu=spec.nu,
                               workers=0, convention=spec.convention).to_c()

    def step_device(o=oc):
        ctx.check(lib.cisdc_gpu_integrate_device(ctx.h, C.c_void_p(d_phi0.data_ptr()), n, C.byref(o),
                                                 C.c_void_p(d_out.data_ptr()), C.byref(rep), _abi.dptr(incs)))
        return rep.counters.newton_iterations

    # FP64 peak (roofline denominator for the Newton/LU kernel; not in MEASURED_PEAKS.json)
    pk_fma, pk_mul = C.c_double(), C.c_double()
    lib.cisdc_gpu_fp64_peak(C.byref(pk_fma), C.byref(pk_mul))

    for _ in range(args.warmup):
        step_device()
    # timed region: per-kernel events off (they would add host work per launch on the small,
    # launch-bound configs); launches are counted regardless
    lib.cisdc_gpu_kernel_times(ctx.h, None, None, None, 0, 1)  # reset
    lib.cisdc_gpu_device_time_ms(ctx.h, 1)
    newton = 0
    rexit0 = lib.cisdc_gpu_newton_residual_exits(ctx.h)
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            newton += step_device()
        torch.cuda.synchronize()
    barrier(ws)
    newton_rexits = lib.cisdc_gpu_newton_residual_exits(ctx.h) - rexit0
    # the same FP64 probe again right after the timed steps: the board is hot and at the clock the
    # Newton kernel ran at (sustained denominator; the one above ran cold, at boost)
    pk_fma_s, pk_mul_s = C.c_double(), C.c_double()
    lib.cisdc_gpu_fp64_peak(C.byref(pk_fma_s), C.byref(pk_mul_s))
    dev_ms = lib.cisdc_gpu_device_time_ms(ctx.h, 1)
    launches = int(lib.cisdc_gpu_launch_count(ctx.h))  # our kernels launched in the timed region
    tmax = max_over_ranks(ws, dev_ms)

    # the same K steps again with live CUDA-event timing of every launch, per kernel class, on the
    # stream each kernel is launched on (roofline + breakdown)
    lib.cisdc_gpu_kernel_times(ctx.h, None, None, None, 0, 1)
    lib.cisdc_gpu_set_timing(ctx.h, 1)
    for _ in range(args.steps):
        step_device(oc1)
    torch.cuda.synchronize()
    inst_ms = lib.cisdc_gpu_device_time_ms(ctx.h, 1)
    ms = (C.c_double * 16)()
    by = (C.c_double * 16)()
    cnt = (C.c_longlong * 16)()
    ncls = lib.cisdc_gpu_kernel_times(ctx.h, ms, by, cnt, 16, 1)
    lib.cisdc_gpu_set_timing(ctx.h, 0)
    updates_per_step = n * spec.M * spec.n_sweeps
    value = ws * updates_per_step * args.steps / (tmax * 1e-3)

    # e2e: host pinned buffers through the C-ABI, copies inside every step
    h_phi0 = torch.from_numpy(spec.phi0).pin_memory()
    h_out = torch.empty_like(h_phi0).pin_memory()
    for _ in range(1):
        ctx.check(lib.cisdc_gpu_integrate(ctx.h, C.cast(h_phi0.data_ptr(), C.POINTER(C.c_double)), n, C.byref(oc),
                                          C.cast(h_out.data_ptr(), C.POINTER(C.c_double)), C.byref(rep),
                                          _abi.dptr(incs)))
    lib.cisdc_gpu_device_time_ms(ctx.h, 1)
    barrier(ws)
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.check(lib.cisdc_gpu_integrate(ctx.h, C.cast(h_phi0.data_ptr(), C.POINTER(C.c_double)), n, C.byref(oc),
                                          C.cast(h_out.data_ptr(), C.POINTER(C.c_double)), C.byref(rep),
                                          _abi.dptr(incs)))
    wall = time.perf_counter() - wall0
    e2e_ms = max_over_ranks(ws, lib.cisdc_gpu_device_time_ms(ctx.h, 1))
    e2e_value = ws * updates_per_step * args.steps / (e2e_ms * 1e-3)

    # roofline of the dominant kernel class
    hbm, hbm_src = measured_peaks()
    classes = []
    for c in range(ncls):
        if cnt[c] == 0:
            continue
        classes.append({"kernel": lib.cisdc_gpu_kernel_class_name(c).decode(), "ms": ms[c], "launches": int(cnt[c]),
                        "share": ms[c] / max(sum(ms[:ncls]), 1e-30),
                        "gbs": (by[c] / (ms[c] * 1e-3) / 1e9) if ms[c] > 0 else None})
    dom = max(classes, key=lambda x: x["ms"])
    cell_solves = desc.ncell * spec.M * spec.n_sweeps * args.steps * (spec.nu if scheme == 2 else 1)
    sparse = os.environ.get("CISDC_RTC", "1") != "0"  # the specialised kernel runs the static-pattern LU
    # the reaction kernel's algorithmic work: the Newton trips and the F_R evaluation of every result
    newton_flops = roofline.newton_work(desc, newton, newton - newton_rexits, sparse=sparse,
                                        cell_solves=cell_solves)
    # FP64 denominator at the clock the timed steps ran at: the burst DMUL/DADD peak (measured cold,
    # at the boost clock) scaled by the median SM clock sampled during the timed steps (the FP64 pipe's
    # rate is proportional to the clock; the burst probe reaches 99% of 64 lanes x 148 SMs x f_max).
    # The probe re-run right after the timed steps (pk_mul_s) is reported beside it: it runs at
    # whatever clock the board has recovered to, so it is a noisier estimate of the same thing.
    clk_pre = clk.summary()
    f_run, f_max = clk_pre.get("sm_mhz"), clk_pre.get("sm_max_mhz")
    clock_scale = (f_run / f_max) if (f_run and f_max) else 1.0
    pk_mul_run = pk_mul.value * min(clock_scale, 1.0)
    # CISDCQ with the fused kernel: R(m)'s Newton solve of nodes 1 .. M-1 runs inside k_react_next (class
    # react_newton_rhs, HBM-bound: it also assembles D(m+1)'s right-hand side), node M's in the stand-alone
    # k_react (class react_newton); the analytic Newton work is apportioned by cell solves
    names = {c["kernel"] for c in classes}
    newton_share = {"react_newton": 1.0}
    if "react_newton_rhs" in names:
        newton_share = {"react_newton": 1.0 / spec.M, "react_newton_rhs": (spec.M - 1.0) / spec.M}
    if dom["kernel"] == "react_newton" and desc.nspecies >= 9:
        achieved = newton_share["react_newton"] * newton_flops / (dom["ms"] * 1e-3) / 1e12
        # The kernel's arithmetic is the reference's no-FMA operation sequence (bit parity), i.e.
        # DADD / DMUL, one flop per FP64 pipe slot: its attainable peak is the measured DMUL/DADD
        # issue rate; the DFMA rate (two flops per slot) is listed beside it.
        roof = {"bound": "fp64", "kernel": dom["kernel"], "achieved": achieved, "peak": pk_mul_run,
                "unit": "TFLOP/s", "frac": achieved / pk_mul_run,
                "peak_source": "measured DMUL/DADD chain peak on this GPU (cisdc_gpu_fp64_peak, burst at the "
                               "boost clock) x the median SM clock of the timed steps / the max clock",
                "peak_burst": pk_mul.value, "frac_of_burst_peak": achieved / pk_mul.value,
                "peak_after_run": pk_mul_s.value, "frac_of_peak_after_run": achieved / pk_mul_s.value,
                "peak_dfma": pk_fma.value, "frac_of_dfma_peak": achieved / pk_fma.value, "traffic": None,
                "work": f"{newton} Newton trips ({newton - newton_rexits} with a Jacobian solve), "
                        f"analytic {newton_flops:.3e} FP64 flops"}
    else:
        achieved = dom["gbs"]
        roof = {"bound": "hbm", "kernel": dom["kernel"], "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "peak_source": hbm_src, "traffic": None}
    # per-class rooflines (HBM classes against the measured copy bandwidth) and the committed ncu
    # capture of each class (DRAM bytes per launch, FP64 pipe utilisation)
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    ncu = {}
    if os.path.exists(prof):
        with open(prof) as f:
            ncu = json.load(f)
    if roof["kernel"] in ncu:
        roof["traffic"] = ncu[roof["kernel"]].get("dram_bytes")
        roof["traffic_source"] = ncu[roof["kernel"]].get("source")
    per_class = []
    for c in classes:
        e = {"kernel": c["kernel"], "share": c["share"], "achieved_gbs": c["gbs"], "hbm_frac": (c["gbs"] or 0) / hbm}
        if c["kernel"] in ncu:
            e["ncu"] = {k: ncu[c["kernel"]].get(k) for k in ("dram_pct", "fp64_pipe_pct", "l1_pct")}
        if c["kernel"] in newton_share and desc.nspecies >= 9:
            e["fp64_tflops"] = newton_share[c["kernel"]] * newton_flops / (c["ms"] * 1e-3) / 1e12
            e["fp64_work_share"] = newton_share[c["kernel"]]
            e["fp64_frac_dmul_dadd_peak"] = e["fp64_tflops"] / pk_mul_run
            e["fp64_frac_peak_after_run"] = e["fp64_tflops"] / pk_mul_s.value
            e["fp64_frac_burst_peak"] = e["fp64_tflops"] / pk_mul.value
        per_class.append(e)

    if rank == 0:
        line = {
            "metric": "cell-species-node updates/s per SDC sweep (FP64)",
            "value": value, "unit": "updates/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tmax / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded BASELINE config generator, problems.py)",
            "config": dict(workload_config(args.config, spec, scheme, workers),
                           parallelism=f"replicas x{ws}"),
            "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "ms_per_step": e2e_ms / args.steps, "wall_s": wall},
            "gpu_launches": launches,
            "roofline": roof,
            "rooflines": sorted(per_class, key=lambda x: -x["share"]),
            "kernels": sorted(classes, key=lambda x: -x["ms"]),
            "kernels_pass": {"ms_per_step": inst_ms / args.steps, "workers": 0,
                             "note": "per-kernel CUDA-event pass, same K steps, one stream"},
            "end_to_end_hbm": {"algorithmic_bytes_per_sweep": 8.0 * n * (7 * spec.M + 4),
                               "achieved_gbs": 8.0 * n * (7 * spec.M + 4) * spec.n_sweeps * args.steps / (tmax * 1e-3) / 1e9},
            "newton_trips_per_cell_solve": newton / max(cell_solves, 1),
            "newton_residual_exit_fraction": newton_rexits / max(cell_solves, 1),
        }
        clk_s = clk.summary()
        line["clocks"] = clk_s
        if ws == 1 and not args.no_cpu_baseline:
            v, t, sample, kind, cores = cpu_reference_sample(args.config, scheme, 0)
            line["cpu_baseline"] = {"value": v, "unit": "updates/s", "cores": cores, "kind": kind, "sample": sample,
                                    "seconds": t, "nproc": os.cpu_count()}
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
