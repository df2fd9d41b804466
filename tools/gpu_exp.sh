#!/bin/bash
# Ad-hoc GPU-box experiment pass (repo root on the box): bash tools/gpu_exp.sh <tag>
TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "tma or hierarchy or ragged or full_size or config_parity or device_looped or cycle_cap" > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.log 2>&1
CISDC_MG_TMA=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c5_cp.log 2>&1
