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


def _link(objs, out):
    newest = max(os.path.getmtime(o) for o in objs)
    if os.path.exists(out) and os.path.getmtime(out) >= newest and not os.environ.get("ZPC_REBUILD"):
        return out
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", out, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-8000:])
        raise RuntimeError(f"link failed for {out}")
    return out


def _nvcc(srcs, out, includes, extra=(), shared=True):
    common = COMMON if shared else [c for c in COMMON if c != "-shared"]
    cmd = [NVCC, *ARCH, *common, *[f"-I{i}" for i in includes], *extra, "-o", out, *srcs]
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
    """Each .cu is compiled to its own object in parallel (-c), then linked into the shared library."""
    from concurrent.futures import ThreadPoolExecutor
    csrc = os.path.join(HERE, "csrc")
    srcs = sorted(os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith(".cu"))
    # ZPC_EXTRA_NVCC / ZPC_LIB_OUT: an alternative build of the same sources (A/B timing via ZPC_LIB)
    out = os.environ.get("ZPC_LIB_OUT") or os.path.join(HERE, "lib", "libzipc.so")
    extra = os.environ.get("ZPC_EXTRA_NVCC", "").split()
    incs = [os.path.join(ROOT, "include"), csrc]
    objdir = os.path.join(os.path.dirname(out), "obj_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(s).replace(".cu", ".o")) for s in srcs]
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        list(ex.map(lambda so: _nvcc([so[0]], so[1], incs, [*extra, "-c"], shared=False), zip(srcs, objs)))
    return _link(objs, out)


def build_gen():
    gsrc = os.path.join(ROOT, "zpc_inputs", "csrc")
    return _nvcc([os.path.join(gsrc, "zpc_gen.cu")], os.path.join(ROOT, "zpc_inputs", "lib", "libzpcgen.so"),
                 [gsrc])


def build_all():
    return build_lib(), build_gen()


if __name__ == "__main__":
    print(build_all())
