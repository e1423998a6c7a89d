"""Timeline of k_score_res, cluster 0 / rank 0 (tuning build: ZPC_LIB=.../libzipc_tune.so ZPC_SCORE_DEBUG=1).

    ZPC_LIB=$PWD/paper_2603_08743_b200/lib/libzipc_tune.so ZPC_SCORE_DEBUG=1 python scripts/res_trace.py [requests]
Per unit (epilogue group of the unit): sweep A (+ reduce), sweep B (+ reduce), exchange wait, merge + sweep C;
per tile (MMA warp): wait for the TMEM slot, wait for the K stage.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_08743_b200 import zipc  # noqa: E402
from paper_2603_08743_b200.batch import batch_of, desc_params, workspace_view  # noqa: E402
from zpc_inputs import CONFIGS  # noqa: E402
from zpc_inputs.device import generate  # noqa: E402

nreq = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = CONFIGS["paper_op"]
if len(sys.argv) > 2:   # another sequence length (slice-placement experiments)
    from zpc_inputs import scaled
    cfg = scaled(cfg, seq_lens=[int(sys.argv[2])] * 64)
w = generate(cfg, 2603, np.arange(nreq))
desc, params = desc_params(w)
b = batch_of(w, desc, params)
for _ in range(3):
    zipc.zpc_plan(desc, params, b)
    zipc.zpc_score(desc, params, b)
torch.cuda.synchronize()
R = nreq
lay = zipc.zpc_workspace_layout_get(desc, params, R)
kept = workspace_view(w, desc, params, "kept", torch.int32, (R * cfg.L * cfg.h_kv, lay.kept_stride))
tt = kept.contiguous().view(torch.int64).reshape(-1).cpu().numpy()
C = int(sys.argv[3]) if len(sys.argv) > 3 else 6
base = None
for rk in range(C):
    t = tt[rk * 8192:(rk + 1) * 8192]
    mma = t[:4096].reshape(-1, 4)[:, :3]
    n = int(np.argmax(mma[:, 0] == 0)) if (mma[:, 0] == 0).any() else len(mma)
    mma = mma[:n]
    if n == 0:
        continue
    if base is None:
        base = mma[0, 0]
    ep = t[4096:].reshape(-1, 8)[:, :5]
    ep = ep[ep[:, 0] != 0]
    d = np.diff(ep, axis=1)
    print(f"rank {rk}: tiles {n} wait slot {np.mean(mma[:,1]-mma[:,0]):.0f} stage {np.mean(mma[:,2]-mma[:,1]):.0f} ns | "
          f"units {len(ep)} A {d[:,0].mean():.0f} B {d[:,1].mean():.0f} xchg {d[:,2].mean():.0f} C {d[:,3].mean():.0f} "
          f"total {(ep[:,4]-ep[:,0]).mean():.0f} ns")
    for i in range(2, 5):
        print("   unit", i, (ep[i] - base))
