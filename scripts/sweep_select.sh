# select stage time: register-resident k_select_reg (default) vs k_select (ZPC_SELECT_REG=0)
for cfg in qwen7b llama8b qwen32b; do for reg in 1 0; do
  r=$(ZPC_SELECT_REG=$reg timeout 200 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stage_ms']['select'], d['value'])" 2>&1 | tail -1)
  echo "cfg=$cfg reg=$reg select_ms,req/s=$r"
done; done
