# A/B of the overlapped two-pass score kernel (ZPC_SCORE_OVL) with bisection knobs (ZPC_SCORE_DEBUG:
# 2 = no epilogue math, 4 = no MMA, 2048 = no K gather); prints the score stage time per combination.
for cfg in ${CFGS:-qwen7b llama8b}; do
for ovl in ${OVLS:-1 0}; do
for dbg in ${DBGS:-0 2 2048 2052}; do
  r=$(ZPC_SCORE_OVL=$ovl ZPC_SCORE_DEBUG=$dbg timeout 200 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_ms']['score'])" 2>&1 | tail -1)
  echo "cfg=$cfg ovl=$ovl dbg=$dbg score_ms=$r"
done; done; done
