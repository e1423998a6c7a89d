#!/bin/bash
# rebuild the production library and the tuning build (-DZPC_TUNING: env knobs, event trace) in parallel
cd "$(dirname "$0")/.."
(ZPC_REBUILD=1 python -c "from paper_2603_08743_b200 import build as b; b.build_lib()" 2>&1 | grep -E "error" | head -20) &
(ZPC_REBUILD=1 ZPC_LIB_OUT=$PWD/paper_2603_08743_b200/lib/libzipc_tune.so ZPC_EXTRA_NVCC="-DZPC_TUNING" python -c "from paper_2603_08743_b200 import build as b; b.build_lib()" 2>&1 | grep -E "error" | head -20) &
wait
