#!/bin/bash
# Quick A/B on the GPU box: targeted GPU tests, then the default bench with and without the knobs under test.
TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "tma or tiled_3d or full_size or config_parity" > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.log 2>&1
CISDC_EVAL_TMA=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c5_evalcp.log 2>&1
CISDC_EVAL_TMA=0 CISDC_MG_TMA=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c5_cp.log 2>&1
