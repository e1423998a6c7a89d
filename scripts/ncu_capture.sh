# ncu --set full captures of the dominant kernels at the bench's exact launches (qwen7b: k_score_coop, k_select_reg,
# k_compact; paper_op: k_score_res, k_red_umma) -> traffic records for bench.py. Run on the GPU box:
#   gpurun -- bash scripts/ncu_capture.sh
O=gpurun_out
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_score|k_compact|k_select" -c 3 \
  -o $O/prof_full -f python scripts/profile_step.py --requests 64 > $O/prof_full.log 2>&1
python scripts/ncu_to_traffic.py $O/prof_full.ncu-rep "ncu --set full --import-source on --clock-control none -k regex:'k_score|k_compact|k_select' -c 3 python scripts/profile_step.py --requests 64 (the bench's qwen7b batch)" $O/traffic.json > /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_score_res|k_red_umma|k_compact" -c 3 \
  -o $O/prof_po -f python scripts/profile_step.py --config paper_op --requests 4 --redundancy > $O/prof_po.log 2>&1
python scripts/ncu_to_traffic.py $O/prof_po.ncu-rep "ncu --set full --import-source on --clock-control none -k regex:'k_score_res|k_red_umma|k_compact' -c 3 python scripts/profile_step.py --config paper_op --requests 4 --redundancy" $O/traffic_paper_op.json > /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_score_tc" -c 1 \
  -o $O/prof_lse -f python scripts/profile_step.py --requests 64 --lse-input > $O/prof_lse.log 2>&1
python scripts/ncu_to_traffic.py $O/prof_lse.ncu-rep "ncu --set full -k regex:k_score_tc -c 1 python scripts/profile_step.py --requests 64 --lse-input" $O/traffic_lse.json > /dev/null
ls -la $O/*.json
