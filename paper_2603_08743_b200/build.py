"""Build libzipc.so (the product, sm_100a only) and libzpcgen.so (the input generator) in-tree.

    python -m paper_2603_08743_b200.build        # or __graft_entry__.build()
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
          "-Xptxas", "-v"]


def _nvcc(srcs, out, includes, extra=()):
    cmd = [NVCC, *ARCH, *COMMON, *[f"-I{i}" for i in includes], *extra, "-o", out, *srcs]
    newest = max(os.path.getmtime(s) for s in srcs + [os.path.join(i, f) for i in includes
                                                      for f in os.listdir(i) if f.endswith(".h")])
    if os.path.exists(out) and os.path.getmtime(out) >= newest and not os.environ.get("ZPC_REBUILD"):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = out + ".buildlog"
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-8000:])
        raise RuntimeError(f"nvcc failed for {out} (see {log})")
    return out


def build_lib():
    csrc = os.path.join(HERE, "csrc")
    srcs = sorted(os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith(".cu"))
    # ZPC_EXTRA_NVCC / ZPC_LIB_OUT: an alternative build of the same sources (A/B timing via ZPC_LIB)
    out = os.environ.get("ZPC_LIB_OUT") or os.path.join(HERE, "lib", "libzipc.so")
    extra = os.environ.get("ZPC_EXTRA_NVCC", "").split()
    return _nvcc(srcs, out, [os.path.join(ROOT, "include"), csrc], extra)


def build_gen():
    gsrc = os.path.join(ROOT, "zpc_inputs", "csrc")
    return _nvcc([os.path.join(gsrc, "zpc_gen.cu")], os.path.join(ROOT, "zpc_inputs", "lib", "libzpcgen.so"),
                 [gsrc])


def build_all():
    return build_lib(), build_gen()


if __name__ == "__main__":
    print(build_all())
