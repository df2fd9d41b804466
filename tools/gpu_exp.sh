#!/bin/bash
TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "hierarchy or config_parity or full_size or cycle_cap or device_looped" > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
for c in c3 c4; do
timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.log 2>&1
CISDC_MG_COARSE=1 timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_${c}_cta.log 2>&1
done
