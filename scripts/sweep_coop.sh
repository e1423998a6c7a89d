#!/bin/bash
# A/B sweep of the cooperative score kernel's tuning knobs (tuning build, ZPC_LIB) on the qwen7b bench.
#   scripts/sweep_coop.sh "KT DELTA HINTS" ...
export ZPC_LIB=$PWD/paper_2603_08743_b200/lib/libzipc_${LIBV:-tune}.so
CFG=${CFG:-qwen7b}
for s in "$@"; do
  set -- $s
  out=$(ZPC_COOP_KT=$1 ZPC_COOP_DELTA=$2 ZPC_COOP_HINTS=$3 ZPC_COOP_DEBUG=${4:-0} timeout 120 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "kt=$1 delta=$2 hints=$3 dbg=${4:-0} $(python3 -c "import json,sys; d=json.loads(sys.argv[1]); print('score_ms', d['stage_ms']['score'], 'value', round(d['value']))" "$out" 2>&1 | tail -1)"
done
