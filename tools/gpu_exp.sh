#!/bin/bash
# Ad-hoc GPU-box experiment pass (repo root on the box): bash tools/gpu_exp.sh <tag>
TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
for c in c1 c2; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/${TAG}_bench_$c.log 2>&1
  CISDC_STEP_GRAPH=0 timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/${TAG}_bench_${c}_nograph.log 2>&1
  timeout 300 python bench.py --config $c --scheme 0 --no-cpu-baseline --steps 20 > gpurun_out/${TAG}_bench_${c}_misdc.log 2>&1
done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.log 2>&1
