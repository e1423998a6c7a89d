"""Benchmark / test harness pieces that are neither product nor oracle.

window_lse_from_two_pass stands in for a decode engine's saved softmax normalisers (the NEXT-4 input of
ZPC_F_LSE_INPUT): it runs the library's own two-pass score stage once, untimed, and converts the log2-domain LSE
workspace region into the natural-log [L][M][w][h_q] layout the ABI takes. Parity tests never trust it: the
sampled units are checked against the oracle's own exact normalisers.
"""
import torch

from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params, workspace_view


def window_lse_from_two_pass(w, flags=0):
    """NEXT-4 input for benchmarks and full-size tests: the fp32 [L][M][w][h_q] natural-log window
    normalisers a decode engine would hold, produced by one two-pass zpc_plan + zpc_score call (its
    LSE workspace region is [R][L][h_kv][w][G], log2 domain) and scattered to the query slots.
    Leaves w.status reset; w.workspace is reused."""
    cfg, lay = w.cfg, w.layout
    desc, params = desc_params(w, flags=flags)
    b = batch_of(w, desc, params)
    zipc.zpc_plan(desc, params, b)
    zipc.zpc_score(desc, params, b)
    R, G = int(w.seq_lens.numel()), cfg.h_q // cfg.h_kv
    lse2 = workspace_view(w, desc, params, "lse", torch.float32, (R, cfg.L, cfg.h_kv, cfg.w, G))
    nat = (lse2 / 1.4426950408889634).permute(1, 0, 3, 2, 4).reshape(cfg.L, R, cfg.w, cfg.h_q)
    out = torch.zeros((cfg.L, lay.M, cfg.w, cfg.h_q), dtype=torch.float32, device=w.k.device)
    out[:, w.q_slots.long()] = nat
    torch.cuda.synchronize()
    w.status.fill_(12345)
    return out
