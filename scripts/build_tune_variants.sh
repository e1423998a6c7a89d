#!/bin/bash
# tuning builds of libzipc with extra defines, in parallel: scripts/build_tune_variants.sh NAME "DEFS" [NAME "DEFS" ...]
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  (ZPC_REBUILD=1 ZPC_LIB_OUT=$PWD/paper_2603_08743_b200/lib/libzipc_$name.so ZPC_EXTRA_NVCC="-DZPC_TUNING $defs" python -c "from paper_2603_08743_b200 import build as b; b.build_lib()" 2>&1 | grep -E " error" | head -5) &
done
wait
