"""Debug timeline of the score kernel's ring (ZPC_SCORE_DEBUG bit 0 = record, CTA 0, 512 steps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params
from zpc_inputs import CONFIGS
from zpc_inputs.device import generate
w = generate(CONFIGS["qwen7b"], 2603, np.arange(int(sys.argv[1]) if len(sys.argv) > 1 else 8))
desc, params = desc_params(w)
b = batch_of(w, desc, params)
zipc.zpc_plan(desc, params, b)
for _ in range(2):
    zipc.zpc_score(desc, params, b)
torch.cuda.synchronize()
lay = zipc.zpc_workspace_layout_get(desc, params, int(w.seq_lens.numel()))
ts = w.workspace[lay.kept:lay.kept + 512 * 32].view(torch.int64).view(512, 4).cpu().numpy()
t0 = ts[0, 0]
print("step  issue   full(MMA)  accfull(epi)   [us rel. to first issue]; lat=full-issue")
for g in list(range(0, 12)) + list(range(60, 72)) + list(range(200, 206)):
    iss, fu, af = (ts[g, :3] - t0) / 1e3
    print(f"{g:4d} {iss:9.2f} {fu:9.2f} {af:9.2f}   lat={fu-iss:7.2f}")
d = np.diff(ts[10:500, 2]) / 1e3
print("median step (epilogue acc_full spacing) us:", np.median(d), "mean", d.mean())
print("median issue->full latency us:", np.median((ts[10:500, 1] - ts[10:500, 0]) / 1e3))
wt = w.workspace[lay.kept + 4096 * 8:lay.kept + 4096 * 8 + 256 * 16 * 8].view(torch.int64).view(256, 16).cpu().numpy()
print("per-warp issue start / end (us rel. to warp-0 start), steps 100..104:")
for g in range(100, 105):
    st = (wt[g, :8] - wt[g, 0]) / 1e3
    en = (wt[g, 8:] - wt[g, 0]) / 1e3
    print(g, "start", np.round(st, 2), "end", np.round(en, 2), " full at", round((ts[g, 1] - wt[g, 0]) / 1e3, 2))
af = ts[:512, 2] / 1e3
d = np.diff(af)
# C=1: 128 steps per unit (64 pass-1, 64 pass-2)
p1 = [d[k] for k in range(10, 500) if (k % 128) < 63]
p2 = [d[k] for k in range(10, 500) if 64 <= (k % 128) < 127]
print("median pass-1 step us:", np.median(p1), " pass-2 step us:", np.median(p2))
