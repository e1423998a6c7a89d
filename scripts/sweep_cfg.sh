# score stage time per config (default build; env in ENV)
for cfg in ${CFGS:-qwen7b llama8b qwen32b}; do
  r=$(timeout 200 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_ms']['score'], d['value'])" 2>&1 | tail -1)
  echo "cfg=$cfg score_ms,req/s=$r"
done
