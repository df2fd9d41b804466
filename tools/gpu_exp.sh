#!/bin/bash
TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
timeout 300 python bench.py > gpurun_out/${TAG}_bench_c5.log 2>&1
timeout 300 python bench.py --scheme 1 --no-cpu-baseline --steps 3 > gpurun_out/${TAG}_bench_c5m.log 2>&1
timeout 300 python bench.py --scheme 0 --no-cpu-baseline --steps 3 > gpurun_out/${TAG}_bench_c5d.log 2>&1
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/${TAG}_bench_c4.log 2>&1
timeout 300 python bench.py --config c4 --scheme 0 --no-cpu-baseline > gpurun_out/${TAG}_bench_c4d.log 2>&1
