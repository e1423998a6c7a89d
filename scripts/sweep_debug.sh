for mode in "" "--lse-input"; do
for dbg in 0 2 4 6 256 262 2048; do
  r=$(ZPC_SCORE_DEBUG=$dbg timeout 200 python bench.py --no-cpu-baseline --no-e2e --steps 5 $mode 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_ms']['score'])" 2>&1 | tail -1)
  echo "mode=$mode dbg=$dbg score_ms=$r"
done; done
