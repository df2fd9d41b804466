#!/bin/bash
# Quick A/B on the GPU box: the default bench against the knobs under test (no CPU baseline leg).
TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.log 2>&1
for z in 64 128 16; do
CISDC_ZCHUNK=$z timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c5_z$z.log 2>&1
done
CISDC_ZCHUNK=64 timeout 600 python -m pytest tests -m gpu -q -x -k "tma or tiled_3d or full_size" > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
