#!/bin/bash
# Checked build (device-side bounds assertions, -DZPC_CHECKS) + the whole GPU suite against it: the stand-in for
# compute-sanitizer memcheck, which this GPU pool does not offer. Run on the GPU box:
#   gpurun -- bash scripts/checked_suite.sh      (log: gpurun_out/checked_suite.log)
cd "$(dirname "$0")/.."
ZPC_REBUILD=1 ZPC_LIB_OUT=$PWD/paper_2603_08743_b200/lib/libzipc_checked.so ZPC_EXTRA_NVCC="-DZPC_CHECKS" \
  python -c "from paper_2603_08743_b200 import build as b; b.build_lib()" || exit 1
mkdir -p gpurun_out
ZPC_LIB=$PWD/paper_2603_08743_b200/lib/libzipc_checked.so timeout 3000 python -m pytest tests -m gpu -q -x \
  > gpurun_out/checked_suite.log 2>&1
echo "checked suite rc=$?"; tail -3 gpurun_out/checked_suite.log
