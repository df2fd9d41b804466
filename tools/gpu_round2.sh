#!/bin/bash
# Shorter GPU-box pass: GPU tests, default bench, ncu launch list + hot-kernel captures, per-config lines.
TAG=${1:-r2p}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
timeout 400 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.log 2>&1
timeout 1200 bash profiles/run_ncu.sh ${TAG} c5 > gpurun_out/${TAG}_ncu.log 2>&1
timeout 2400 bash tools/bench_configs.sh ${TAG}
