"""Per-step critical-path timeline of k_score_tc (debug bit 1, CTA 0): epilogue and MMA stamps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params
from zpc_inputs import CONFIGS
from zpc_inputs.device import generate
w = generate(CONFIGS["qwen7b"], 2603, np.arange(int(sys.argv[1]) if len(sys.argv) > 1 else 16))
desc, params = desc_params(w)
b = batch_of(w, desc, params)
zipc.zpc_plan(desc, params, b)
zipc.zpc_score(desc, params, b)
torch.cuda.synchronize()
lay = zipc.zpc_workspace_layout_get(desc, params, int(w.seq_lens.numel()))
raw = w.workspace[lay.kept:lay.kept + 20480 * 8].view(torch.int64).cpu().numpy()
E = raw[8192:8192 + 4096].reshape(1024, 4)[:, :3] / 1e3
M = raw[16384:16384 + 4096].reshape(1024, 4) / 1e3
t0 = M[0, 0]
npass = 32 if len(sys.argv) < 3 else int(sys.argv[2])   # steps per pass per CTA (C=2: 32)
print("step | MMA: wait_acce  wait_full  issued | EPI: wait_start  got_acc  done   (us)")
for g in list(range(130, 142)):
    print(f"{g:4d} P{1 + ((g % (2*npass)) >= npass)} | {M[g,0]-t0:8.2f} {M[g,1]-t0:8.2f} {M[g,2]-t0:8.2f} {M[g,3]-t0:8.2f} | {E[g,0]-t0:8.2f} {E[g,1]-t0:8.2f} {E[g,2]-t0:8.2f}")
sl = slice(64, 900)
epi_wait = E[sl, 1] - E[sl, 0]
epi_work = E[sl, 2] - E[sl, 1]
mma_wait_acce = M[sl, 1] - M[sl, 0]
mma_wait_full = M[sl, 2] - M[sl, 1]
p1 = np.array([(g % (2 * npass)) < npass for g in range(64, 900)])
for name, x in [("epi wait", epi_wait), ("epi work", epi_work), ("mma wait acc_empty", mma_wait_acce), ("mma wait full", mma_wait_full)]:
    print(f"{name:20s} P1 median {np.median(x[p1]):6.3f}  P2 median {np.median(x[~p1]):6.3f}  us")
