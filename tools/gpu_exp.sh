#!/bin/bash
# Ad-hoc GPU-box experiment pass (repo root on the box): bash tools/gpu_exp.sh <tag>
TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
timeout 300 python bench.py > gpurun_out/${TAG}_bench_c5.log 2>&1
timeout 1200 bash profiles/run_ncu.sh ${TAG} c5 > gpurun_out/${TAG}_ncu.log 2>&1
