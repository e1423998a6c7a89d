"""Event timeline of k_score_coop's pair 0 (tuning build: ZPC_LIB=.../libzipc_tune.so, ZPC_COOP_TRACE=1).

    ZPC_LIB=$PWD/paper_2603_08743_b200/lib/libzipc_tune.so ZPC_COOP_TRACE=1 python scripts/coop_trace.py
Prints where the MMA issuer of pair 0 waits: per step, (top -> stage full) and (full -> accumulator / aug
ready), summed by step kind, plus the combiner's counter waits.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_08743_b200 import zipc  # noqa: E402
from paper_2603_08743_b200.batch import batch_of, desc_params  # noqa: E402
from zpc_inputs import CONFIGS  # noqa: E402
from zpc_inputs.device import generate  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "qwen7b"]
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 64
w = generate(cfg, 2603, np.arange(nreq))
desc, params = desc_params(w)
b = batch_of(w, desc, params)
for _ in range(2):
    zipc.zpc_plan(desc, params, b)
    zipc.zpc_score(desc, params, b)
torch.cuda.synchronize()
buf = (ctypes.c_uint32 * 49152)()
rc = zipc.lib().zpc_debug_trace_copy(ctypes.byref(buf), ctypes.c_size_t(49152 * 4))
assert rc == 0, "not a tuning build"
t = np.frombuffer(buf, dtype=np.uint32).astype(np.int64)
mma = t[:32768].reshape(-1, 4)
n = int(np.argmax(mma[:, 3] == 0)) if (mma[:, 3] == 0).any() else len(mma)
mma = mma[:n]
kind = mma[:, 1] & 1
first = (mma[:, 1] >> 1) & 1
top = mma[:, 0]
def d(a, b):
    return (b - a) % (1 << 32)
wfull = d(top, mma[:, 1])
wready = d(mma[:, 1], mma[:, 2])
issue = d(mma[:, 2], mma[:, 3])
gap = np.r_[0, d(mma[:-1, 3], top[1:])]
total = d(top[0], mma[-1, 3])
clk_span, ns_span = d(t[49148], t[49150]), d(t[49149], t[49151])
if ns_span > 0:
    print(f"pair 0 MMA loop: {clk_span} clk in {ns_span / 1e3:.1f} us -> SM clock {clk_span / ns_span:.3f} GHz")
print(f"steps {n}  span {total} clk ({total / 1.9e3:.1f} us at 1.9 GHz)  per step {total / n:.0f} clk")
for k, name in [(0, "pass1"), (1, "pass2")]:
    m = kind == k
    print(f"{name}: steps {m.sum():5d}  wait full {wfull[m].mean():7.0f}  wait acc/aug {wready[m].mean():7.0f}  "
          f"issue {issue[m].mean():6.0f}  sched gap {gap[m].mean():6.0f}   (sum full {wfull[m].sum()/total:.1%}, "
          f"ready {wready[m].sum()/total:.1%})")
    mf = m & (first == 1)
    if mf.any():
        print(f"   first tile of a chunk: wait full {wfull[mf].mean():7.0f} ready {wready[mf].mean():7.0f} (n={mf.sum()})")
comb = t[32768:40960].reshape(-1, 4)
nc = int(np.argmax(comb[:, 0] == 0)) if (comb[:, 0] == 0).any() else len(comb)
comb = comb[:nc]
print(f"combiner chunks {nc}: counter wait mean {d(comb[:, 0], comb[:, 1]).mean():.0f} clk, "
      f"to aug written {d(comb[:, 1], comb[:, 2]).mean():.0f} clk")
pub = t[40960:45056].reshape(-1, 2)
npb = int(np.argmax(pub[:, 0] == 0)) if (pub[:, 0] == 0).any() else len(pub)
print(f"pass-1 publish fence+atomic: mean {d(pub[:npb, 0], pub[:npb, 1]).mean():.0f} clk over {npb} chunks")
p1 = t[45056:49152].reshape(-1, 4)
n1 = int(np.argmax(p1[:, 3] == 0)) if (p1[:, 3] == 0).any() else len(p1)
p1 = p1[:n1]
if n1 > 2:
    print(f"pass-1 warp 8, {n1} sub-steps: wait accf {d(p1[:, 0], p1[:, 1]).mean():.0f}  load+release {d(p1[:, 1], p1[:, 2]).mean():.0f}"
          f"  compute {d(p1[:, 2], p1[:, 3]).mean():.0f}  (period {d(p1[:-1, 0], p1[1:, 0]).mean():.0f} clk)")
np.save(os.path.join(ROOT, "gpurun_out", "coop_trace.npy"), t)
