#!/bin/bash
# One GPU-box pass (run from the repo root on the box): GPU tests, the default bench line, ncu captures
# of the C5 hot kernels (TMA walker on, and the cp.async walker for the multigrid sweep), and the
# per-config bench lines.   bash tools/gpu_round.sh <tag>
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputest.log
timeout 400 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 1200 bash profiles/run_ncu.sh ${TAG} c5 > gpurun_out/${TAG}_ncu.log 2>&1
CISDC_MG_TMA=0 timeout 600 bash -c "N=/usr/local/cuda/bin/ncu; \$N --set full --clock-control none --import-source on -k 'regex:k_mg3_pair' -c 4 -f -o /tmp/${TAG}_cpasync python tools/profile_step.py --config c5 --scale 1 > gpurun_out/ncu_${TAG}_cpasync.log 2>&1; \$N -i /tmp/${TAG}_cpasync.ncu-rep --page raw --csv > gpurun_out/${TAG}_c5_mg3cp_raw.csv"
timeout 2400 bash tools/bench_configs.sh ${TAG}
