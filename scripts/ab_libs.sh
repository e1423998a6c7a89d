#!/bin/bash
# interleaved A/B of library builds on one box: scripts/ab_libs.sh ROUNDS lib1.so lib2.so ...  (CFG, EXTRA env)
R=$1; shift
CFG=${CFG:-qwen7b}
for r in $(seq 1 $R); do
  for lib in "$@"; do
    out=$(ZPC_LIB=$PWD/paper_2603_08743_b200/lib/$lib timeout 180 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $EXTRA 2>/dev/null | tail -1)
    echo "$lib $(python3 -c "import json,sys; d=json.loads(sys.argv[1]); print('score_ms', d['stage_ms']['score'], 'value', round(d['value']), 'mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])" "$out" 2>&1 | tail -1)"
  done
done
