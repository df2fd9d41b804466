#!/bin/bash
# Per-config bench lines: every BASELINE config with its own scheme, plus the
# MISDC / MISDCQ / serial-CISDCQ arms of C5.  Run on the GPU box from the repo root:
#   bash tools/bench_configs.sh <tag>      -> gpurun_out/<tag>_configs.jsonl (one JSON line per run)
TAG=${1:-r2}
OUT=gpurun_out/${TAG}_configs.jsonl
mkdir -p gpurun_out
: > $OUT
run() {  # label, bench args...
  local label=$1; shift
  local line
  line=$(timeout 600 python bench.py --no-cpu-baseline "$@" 2> gpurun_out/${TAG}_cfg_${label}.err | grep '^{' | tail -1)
  if [ -n "$line" ]; then
    python -c "import json,sys; d=json.loads(sys.argv[1]); d['label']=sys.argv[2]; d['argv']=sys.argv[3:]; print(json.dumps(d))" "$line" "$label" "$@" >> $OUT
  else
    echo "{\"label\": \"$label\", \"failed\": true}" >> $OUT
  fi
}
run c1 --config c1 --steps 20 --warmup 5
run c2 --config c2 --steps 10 --warmup 3
run c3 --config c3 --steps 5 --warmup 3
run c4 --config c4 --steps 5 --warmup 3
run c5 --config c5 --steps 5 --warmup 3
run c5_misdc --config c5 --scheme 0 --steps 3 --warmup 3
run c5_misdcq --config c5 --scheme 1 --steps 3 --warmup 3
run c5_cisdcq_serial --config c5 --workers 0 --steps 3 --warmup 3
run c1_misdc --config c1 --scheme 0 --steps 20 --warmup 5
run c2_misdc --config c2 --scheme 0 --steps 10 --warmup 3
run c3_misdc --config c3 --scheme 0 --steps 5 --warmup 3
run c4_misdc --config c4 --scheme 0 --steps 5 --warmup 3
run c5_imexq --config c5 --scheme 3 --steps 2 --warmup 1
run c3_imexq --config c3 --scheme 3 --steps 2 --warmup 1
