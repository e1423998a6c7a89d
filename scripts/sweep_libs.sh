# score stage time per alternative build (ZPC_LIB) x env setting, qwen7b unless CFG is set
run() { timeout 200 python bench.py --config ${CFG:-qwen7b} --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_ms']['score'])" 2>&1 | tail -1; }
for lib in ${LIBS:-default}; do
  L=""; [ "$lib" != default ] && L=paper_2603_08743_b200/lib/alt/$lib.so
  for env in ${ENVS:-X=0}; do
    for dbg in ${DBGS:-0}; do
      echo "lib=$lib env=$env dbg=$dbg score_ms=$(export $env ZPC_LIB=$L ZPC_SCORE_DEBUG=$dbg; run)"
    done
  done
done
