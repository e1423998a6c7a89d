"""Per-step critical-path timeline of k_score_tc (debug bit 1, CTA 0): epilogue and MMA stamps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params
from zpc_inputs import CONFIGS
from zpc_inputs.device import generate
w = generate(CONFIGS["qwen7b"], 2603, np.arange(int(sys.argv[1]) if len(sys.argv) > 1 else 16))
LSE = os.environ.get("TL_LSE") == "1"    # NEXT-4 single-pass mode: every step is a pass-2 step
if LSE:
    from zpc_harness import window_lse_from_two_pass
    w.window_lse = window_lse_from_two_pass(w)
desc, params = desc_params(w, lse_input=LSE)
b = batch_of(w, desc, params)
zipc.zpc_plan(desc, params, b)
zipc.zpc_score(desc, params, b)
torch.cuda.synchronize()
lay = zipc.zpc_workspace_layout_get(desc, params, int(w.seq_lens.numel()))
raw = w.workspace[lay.kept:lay.kept + 49152 * 8].view(torch.int64).cpu().numpy()
E = raw[8192:8192 + 4096].reshape(1024, 4)[:, :3] / 1e3
M = raw[16384:16384 + 4096].reshape(1024, 4) / 1e3
t0 = M[0, 0]
npass = 32 if len(sys.argv) < 3 else int(sys.argv[2])   # steps per pass per CTA (C=2: 32)
if LSE:
    npass = 10 ** 9   # label everything P2
print("step | MMA: wait_acce  wait_full  issued | EPI: wait_start  got_acc  done   (kcycles)")
for g in list(range(156, 166)) + list(range(188, 198)):
    print(f"{g:4d} P{1 + ((g % (2*npass)) >= npass)} | {M[g,0]-t0:8.2f} {M[g,1]-t0:8.2f} {M[g,2]-t0:8.2f} {M[g,3]-t0:8.2f} | {E[g,0]-t0:8.2f} {E[g,1]-t0:8.2f} {E[g,2]-t0:8.2f}")
sl = slice(64, 900)
epi_wait = E[sl, 1] - E[sl, 0]
epi_work = E[sl, 2] - E[sl, 1]
mma_wait_acce = M[sl, 1] - M[sl, 0]
mma_wait_full = M[sl, 2] - M[sl, 1]
p1 = np.array([(g % (2 * npass)) < npass for g in range(64, 900)]) if not LSE else np.zeros(836, bool)
for name, x in [("epi wait", epi_wait), ("epi work", epi_work), ("mma wait acc_empty", mma_wait_acce), ("mma wait full", mma_wait_full)]:
    print(f"{name:20s} P1 median {np.median(x[p1])*1e3:6.0f}  P2 median {np.median(x[~p1])*1e3:6.0f}  cycles")

# distribution of epilogue step work (all steps), per pass
for nm, sel in (("P1", p1), ("P2", ~p1)):
    if not sel.any():
        continue
    x = epi_work[sel] * 1e3
    print(nm, "work percentiles (cycles) 10/25/50/75/90:", [int(np.percentile(x, q)) for q in (10, 25, 50, 75, 90)])

# per-unit accounting: steps of a unit vs the unit's wall span (first epilogue start .. last done)
spans = []
for un in (range(2, 12) if not LSE else []):
    g0, g1 = un * 2 * npass, (un + 1) * 2 * npass - 1
    spans.append((E[g1, 2] - E[g0, 0]) * 1e3)
if spans:
    print("unit span (cycles) median", int(np.median(spans)), " sum of step work median",
          int(np.median([np.sum(epi_work[(un * 2 * npass - 64):((un + 1) * 2 * npass - 64)]) * 1e3 for un in range(2, 12)])))

ncta = 148
big = w.workspace[lay.kept:lay.kept + (65536 + ncta * 64) * 8].view(torch.int64).cpu().numpy()
T8 = big[65536:65536 + ncta * 64].reshape(ncta, 8, 8).astype(np.float64)
print("per-warp register timing, mean over CTAs (cycles per step):")
for ew in range(8):
    x = T8[:, ew, :]
    n1 = x[:, 1].sum(); n2 = x[:, 7].sum()
    print(f"  warp {8 + ew} (SMSP {ew % 4}, half {ew // 4}): P1 work {x[:, 0].sum() / n1:6.0f} gap {x[:, 2].sum() / n1:6.0f} | "
          f"P2 ld {x[:, 3].sum() / n2:6.0f} math {x[:, 4].sum() / n2:6.0f} work {x[:, 6].sum() / n2:6.0f} gap {x[:, 5].sum() / n2:6.0f}")
# loader view: step g's loads issued at L[g] (CTA 0, loader thread 0); full at M[g, 2]
L = raw[0:2048].reshape(512, 4)[:, 0] / 1e3
print("step  load_issue  -> full (latency)   MMA step start - load issue (lookahead)   [kcycles]")
for g in list(range(156, 166)) + list(range(188, 196)):
    print(f"{g:4d} P{1 + ((g % (2*npass)) >= npass)} {L[g]-t0:9.2f} {M[g,2]-t0:9.2f} ({M[g,2]-L[g]:5.2f})  {M[g,0]-L[g]:6.2f}")
lat = [(M[g, 2] - L[g]) * 1e3 for g in range(64, 500)]
p1s = [((g % (2 * npass)) < npass) and not LSE for g in range(64, 500)]
print("load->full latency median P1", int(np.median([x for x, f in zip(lat, p1s) if f] or [0])), " P2", int(np.median([x for x, f in zip(lat, p1s) if not f])), "cycles")
LW = raw[4096:4096 + 256 * 16].reshape(256, 16) / 1e3
print("loader warps: start (after stage free) .. end (copies issued) per warp [kcycles rel.], step period")
for g in list(range(180, 192)):
    st = LW[g, 0:4] - t0; en = LW[g, 8:12] - t0
    print(f"{g:4d} P{1 + ((g % (2*npass)) >= npass)} start " + " ".join(f"{x:8.2f}" for x in st) + " | issue dur " + " ".join(f"{x:5.2f}" for x in (en - st)) + f" | full {M[g,2]-t0:8.2f}")
RL = raw[40960:40960 + 2048].reshape(1024, 2) / 1e3
print("relay: step | relay start wait  | accf seen | MMA issued(M3) | epi barrier exit (E1) | epi prev done (E2[g-1])")
for g in list(range(150, 160)) + list(range(176, 184)):
    print(f"{g:4d} P{1 + ((g % (2*npass)) >= npass)} {RL[g,0]-t0:9.2f} {RL[g,1]-t0:9.2f} {M[g,3]-t0:9.2f} {E[g,1]-t0:9.2f} {E[g-1,2]-t0:9.2f}")
