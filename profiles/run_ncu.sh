#!/bin/bash
# ncu recipe for the profiles/ summaries (run on the GPU box from the repo root, one GPU):
#   bash profiles/run_ncu.sh <tag> [config] [scale] [hot|all] [launches]
# 1. launch list (serialised per-launch durations) of one SDC step through the C-ABI
# 2. --set full captures of the hot kernels, exported on the box to CSV (raw metrics, details,
#    source) so that only small files travel back
set -x
TAG=${1:-r1}
CFG=${2:-c5}
SCALE=${3:-1}
N=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
STEP="python tools/profile_step.py --config $CFG --scale $SCALE"
$N --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv $STEP > gpurun_out/ncu_${TAG}_l.log 2>&1
cap() {  # name regex count
  local rep=/tmp/${TAG}_${CFG}_$1
  $N --set full --clock-control none --cache-control ${CACHE:-all} --import-source on -k "regex:$2" -s ${SKIP:-0} -c $3 -f -o $rep $STEP > gpurun_out/ncu_${TAG}_$1.log 2>&1
  $N -i $rep.ncu-rep --page raw --csv > gpurun_out/${TAG}_${CFG}_$1_raw.csv 2>/dev/null
  $N -i $rep.ncu-rep --page details --csv > gpurun_out/${TAG}_${CFG}_$1_details.csv 2>/dev/null
  $N -i $rep.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${CFG}_$1_source.csv 2>/dev/null
  gzip -f gpurun_out/${TAG}_${CFG}_$1_source.csv
}
if [ "${4:-hot}" = "all" ]; then
  # every kernel class of a (small) config: the first ${5:-60} launches, one capture
  cap all ".*" ${5:-60}
else
  cap mg3 "k_mg3_tiled|k_mg3_pair|k_mg3_tma" 4
  cap eval k_eval_ad3 2
  # the second sweep's Newton launches (the first sweep's fields alias node 0): D(2..M)'s rhs rows
  SKIP=6 cap react "^k_react$|^k_react_next$" 6
  cap rhs "^k_rhs$" 2
  cap quad "k_quad|k_mg_update|copy_unswept" 4
fi
ls -la gpurun_out
