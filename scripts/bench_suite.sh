# Round bench suite: every bench line recorded under profiles/ (run on the GPU box via gpurun)
#   gpurun -- bash scripts/bench_suite.sh   (then copy gpurun_out/bench_*.json to profiles/rNN_bench_*.json)
set -x
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --lse-input --no-cpu-baseline > $O/bench_lse.json 2> $O/bench_lse.err
timeout 600 python bench.py --redundancy --no-cpu-baseline > $O/bench_red.json 2> $O/bench_red.err
timeout 600 python bench.py --config paper_op --graph --steps 50 > $O/bench_paper_op.json 2> $O/bench_paper_op.err
timeout 600 python bench.py --config paper_op --graph --steps 50 --redundancy --no-cpu-baseline > $O/bench_paper_op_red.json 2> $O/bench_paper_op_red.err
timeout 600 python bench.py --config paper_op --graph --steps 50 --wave 1 --no-cpu-baseline > $O/bench_paper_op_w1.json 2> $O/bench_paper_op_w1.err
timeout 600 python bench.py --config llama8b --no-cpu-baseline > $O/bench_llama8b.json 2> $O/bench_llama8b.err
timeout 600 python bench.py --config qwen32b --no-cpu-baseline > $O/bench_qwen32b.json 2> $O/bench_qwen32b.err
timeout 600 python bench.py --config prefix --no-cpu-baseline > $O/bench_prefix.json 2> $O/bench_prefix.err
timeout 600 python bench.py --config prefix --lse-input --no-cpu-baseline > $O/bench_prefix_lse.json 2> $O/bench_prefix_lse.err
timeout 600 python bench.py --scaling strong --no-cpu-baseline > $O/bench_strong1.json 2> $O/bench_strong1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_bench.log 2>&1
tail -c 300 $O/bench_*.json
