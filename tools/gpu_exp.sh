#!/bin/bash
# Quick pass on the GPU box: targeted GPU tests, then (optionally) the full GPU suite, smoke() and the default bench.
TAG=${1:-r2x}
SEL=${2:-imexq}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "$SEL" > gpurun_out/${TAG}_gputest_sel.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest_sel.log
if [ "${3:-full}" = "full" ]; then
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_smoke.log
timeout 400 python bench.py > gpurun_out/${TAG}_bench_c5.log 2>&1
fi
