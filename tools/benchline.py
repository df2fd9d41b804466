"""Print the headline numbers and the per-kernel table of bench.py JSON logs (dev helper)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        e2e = d.get("e2e", {}).get("value")
        print(f"{path}: value {d['value']:.4g} {d['unit']}  ms/step {d['ms_per_step']:.2f}  e2e {e2e:.4g}  "
              f"launches {d.get('gpu_launches')}  clocks {d.get('clocks', {}).get('sm_mhz')} "
              f"{d.get('clocks', {}).get('reasons')}")
        steps = d["steps"]
        for k in d.get("kernels", []):
            print(f"   {k['kernel']:14s} {k['ms'] / steps:8.2f} ms/step  {k['launches'] / steps:6.0f} launches  "
                  f"{k.get('gbs', 0):7.0f} GB/s")
