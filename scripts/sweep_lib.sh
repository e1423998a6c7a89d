# A/B of alternative library builds (ZPC_LIB) x score debug masks; prints the score stage time
for lib in "$@"; do
for mode in "" "--lse-input"; do
for dbg in ${DBGS:-0 262}; do
  r=$(ZPC_LIB=$lib ZPC_SCORE_DEBUG=$dbg timeout 200 python bench.py --no-cpu-baseline --no-e2e --steps 5 $mode 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_ms']['score'], d['value'])" 2>&1 | tail -1)
  echo "lib=$(basename $lib) mode=$mode dbg=$dbg score_ms,req/s=$r"
done; done; done
