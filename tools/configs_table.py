"""BASELINE.md section 4 table from the per-config bench lines (tools/bench_configs.sh) and, optionally,
the reference-arm lines of the same box (bench.py --impl reference --config cN).

  python tools/configs_table.py gpurun_out/<tag>_configs.jsonl [gpurun_out/<tag>_ref_*.log ...]
"""
import json
import sys


def lines(path):
    with open(path) as f:
        return [json.loads(x) for x in f if x.startswith("{")]


def main():
    runs = lines(sys.argv[1])
    ref = {}
    for p in sys.argv[2:]:
        for d in lines(p):
            if d.get("impl") == "reference":
                ref[d["config"]["workload"].split(":")[0]] = d
    print("| Config | Scheme (nu, streams) | GPU updates/s | ms / step | e2e updates/s | end-to-end % HBM roofline "
          "| worst kernel (% roofline) | CPU reference updates/s (threads, sample) | SM clock |")
    print("|---|---|---|---|---|---|---|---|---|")
    for d in runs:
        if d.get("failed"):
            print(f"| {d['label']} | failed | | | | | | | |")
            continue
        cfg = d["config"]
        name = cfg["workload"].split(":")[0]
        hbm = d["end_to_end_hbm"]["achieved_gbs"] / d["roofline"]["peak"] if d["roofline"]["unit"] == "GB/s" else \
            d["end_to_end_hbm"]["achieved_gbs"] / 6548.2
        # a class's roofline fraction is its better one (the fused Newton + rhs kernel is HBM-bound with its
        # FP64 work hidden under the loads)
        def frac(r):
            return max(r.get("fp64_frac_dmul_dadd_peak", 0.0), r["hbm_frac"])

        worst = min((r for r in d["rooflines"] if r.get("share", 0) > 0.05 and r.get("hbm_frac")), key=frac,
                    default=None)
        if worst is None:
            ws = "—"
        elif worst.get("fp64_frac_dmul_dadd_peak", 0.0) > worst["hbm_frac"]:
            ws = f"{worst['kernel']} ({100 * worst['fp64_frac_dmul_dadd_peak']:.0f}% FP64)"
        else:
            ws = f"{worst['kernel']} ({100 * worst['hbm_frac']:.0f}% HBM)"
        streams = cfg.get("workers", 0)
        sch = f"{cfg['scheme']} (nu={cfg['nu']}, {'2 streams' if cfg['scheme'] == 'cisdcq' and streams else '1 stream'})"
        r = ref.get(name) if d["label"] == name else None
        cpu = (f"{r['value']:.3g} ({r['cpu_baseline']['cores']} thr, {r['config'].get('sample_scale_per_axis', '')} "
               f"per axis)") if r else "—"
        print(f"| {d['label']} | {sch} | {d['value']:.3g} | {d['ms_per_step']:.3f} | {d['e2e']['value']:.3g} | "
              f"{100 * hbm:.1f}% | {ws} | {cpu} | {d['clocks'].get('sm_mhz')} MHz {d['clocks'].get('reasons')} |")


if __name__ == "__main__":
    main()
