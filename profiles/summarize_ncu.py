#!/usr/bin/env python
"""Summarise the ncu exports of profiles/run_ncu.sh into profiles/<tag>_summary.md and the per-launch
DRAM traffic table profiles/ncu_traffic_<config>.json that bench.py reports as roofline.traffic.

  python profiles/summarize_ncu.py <tag> <config> <dir-with-exports>
"""
import collections
import csv
import json
import os
import sys

# kernel base name -> bench.py kernel class
CLASS = {"k_react": "react_newton", "k_react_next": "react_newton_rhs", "k_eval_ad3_tiled": "eval_ad", "k_eval_ad3_pair": "eval_ad", "k_eval_ad3_tma": "eval_ad",
         "k_eval_ad2_rows": "eval_ad", "k_rhs": "rhs", "k_quad_base": "quad_base", "k_mg3_tiled": "mg_smooth",
         "k_mg3_pair": "mg_smooth", "k_mg3_tma": "mg_smooth", "k_mg2_rows": "mg_smooth", "k_mg_update": "mg_norm",
         "k_mg_copy_unswept": "mg_norm"}

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
]
SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def base_name(k: str) -> str:
    k = k.split("(")[0].replace("void ", "").strip()
    return k.split("<")[0].split("::")[-1]


def load_raw(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for m, _ in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    d[m] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
        out.append(d)
    return out


def launch_list(path):
    agg = collections.OrderedDict()
    for r in csv.reader(open(path)):
        if len(r) < 10 or r[0] == "ID":
            continue
        try:
            v = float(r[-1].replace(",", ""))
        except ValueError:
            continue
        us = v * SCALE.get(r[-2], 1.0)
        k = base_name(r[4]) if len(r) > 4 else "?"
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += us
    return agg


def main():
    tag, cfg, d = sys.argv[1], sys.argv[2], sys.argv[3]
    here = os.path.dirname(os.path.abspath(__file__))
    lines = [f"# ncu summary `{tag}` ({cfg}), from `profiles/run_ncu.sh {tag} {cfg}`", ""]
    ll = os.path.join(d, f"launches_{tag}_{cfg}.csv")
    if os.path.exists(ll):
        agg = launch_list(ll)
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list (one SDC step, `--metrics gpu__time_duration.sum --clock-control none`)", "",
                  "Serialised, cold-cache per-launch durations: compare shares, not absolute times.", "",
                  "| kernel | launches | total ms | us / launch | share |", "|---|---:|---:|---:|---:|"]
        for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| {k} | {n} | {us / 1e3:.2f} | {us / n:.1f} | {100 * us / tot:.1f}% |")
        lines += [f"| **total** | | **{tot / 1e3:.2f}** | | |", ""]
    traffic = {}
    acc = {}
    lines += ["## `--set full` captures", "", "| kernel | " + " | ".join(n for _, n in METRICS) + " | DRAM GB/s |",
              "|---|" + "---:|" * (len(METRICS) + 1)]
    for part in ("react", "eval", "mg3", "rhs", "quad", "rhsd", "all"):
        p = os.path.join(d, f"{tag}_{cfg}_{part}_raw.csv")
        if not os.path.exists(p):
            continue
        seen = set()
        for r in load_raw(p):
            if part == "all":  # one row per distinct kernel (its first capture)
                key = r["kernel"].split("(")[0]
                if key in seen:
                    continue
                seen.add(key)
            t = r.get("gpu__time_duration.sum", 0.0)
            rd, wr = r.get("dram__bytes_read.sum", 0.0), r.get("dram__bytes_write.sum", 0.0)
            cells = []
            for m, _ in METRICS:
                v = r.get(m)
                if v is None:
                    cells.append("")
                elif m == "gpu__time_duration.sum":
                    cells.append(f"{v:.1f} us")
                elif "bytes" in m:
                    cells.append(f"{v / 1e9:.3f} GB")
                else:
                    cells.append(f"{v:.1f}")
            gbs = (rd + wr) / (t * 1e-6) / 1e9 if t else 0.0
            name = r["kernel"].split("(")[0].replace("void ", "")
            lines.append(f"| {name} | " + " | ".join(cells) + f" | {gbs:.0f} |")
            cls = CLASS.get(base_name(r["kernel"]))
            if cls:
                acc.setdefault(cls, []).append({
                    "kernel": name, "dram_bytes": rd + wr, "time_us": t,
                    "dram_pct": r.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                    "fp64_pipe_pct": r.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                    "l1_pct": r.get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                    "part": part})
    # per class: the mean over the captured launches (bench.py's `achieved` is a per-launch mean too)
    for cls, rows in acc.items():
        n = len(rows)
        mean = {k: sum((r[k] or 0.0) for r in rows) / n for k in ("dram_bytes", "time_us", "dram_pct", "fp64_pipe_pct", "l1_pct")}
        mean["kernel"] = rows[0]["kernel"]
        mean["launches_captured"] = n
        mean["source"] = f"profiles/{tag[:2]}/{tag}_{cfg}_{rows[0]['part']}_raw.csv.gz (mean of {n} captured launch(es))"
        traffic[cls] = mean
    lines.append("")
    name = f"{tag}_summary.md" if cfg == "c5" else f"{tag}_{cfg}_summary.md"
    with open(os.path.join(here, name), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(here, f"ncu_traffic_{cfg}.json"), "w") as f:
        json.dump({k: v for k, v in traffic.items()}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
