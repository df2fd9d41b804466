"""Print a compact summary of bench.py JSON lines (development helper, not a test)."""
import json
import sys

for path in sys.argv[1:]:
    lines = [x for x in open(path) if x.startswith("{")]
    if not lines:
        print(path, "NO JSON:", open(path).read()[-1500:])
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline", {})
    print(f"{path}: value={d['value']:.4g} ms/step={d['ms_per_step']:.3f} e2e={d['e2e']['value']:.4g} "
          f"launches={d.get('gpu_launches')} roof={r.get('kernel')} {r.get('achieved', 0):.4g}/{r.get('peak', 0):.4g} "
          f"{r.get('unit')} frac={r.get('frac', 0):.3f} clocks={d.get('clocks', {}).get('sm_mhz')} "
          f"{d.get('clocks', {}).get('reasons')}")
    kp = d.get("kernels_pass")
    if kp:
        print("   kernels pass ms/step", round(kp["ms_per_step"], 3))
    steps = d["steps"]
    for k in d.get("kernels", []):
        print(f"   {k['kernel']:14s} {k['ms'] / steps:9.3f} ms/step {k['launches'] // steps:6d} launches/step "
              f"{1000 * k['ms'] / max(k['launches'], 1):8.1f} us/launch  {k['gbs'] or 0:8.1f} GB/s")
    if "cpu_baseline" in d:
        print("   cpu_baseline", d["cpu_baseline"])
