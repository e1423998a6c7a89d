"""GPU parity of NEXT-4 (ZPC_F_LSE_INPUT): single-pass scoring with the window normalisers supplied
by the caller (PAPER.md:409-411 with the softmax normaliser given).

The normalisers are computed by the fp64 oracle from the definition (oracle.all_window_lse) and
rounded to fp32 -- what a decode attention kernel would hand over. Rules: every §8(c) parity rule
(scores 1e-3 relative, band rule, strict select, bit-exact bytes) against the oracle run with the
SAME normalisers; a perturbed-normaliser case proves the kernel reads the input instead of
recomputing it; the workspace LSE region holds the input in the log2 domain.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params, workspace_view
from zpc_inputs import CONFIGS, make_host_workload, scaled
from zpc_inputs.device import from_host

from helpers import full_check, geometry, gpu_results, snapshot_inputs

pytestmark = pytest.mark.gpu

CASES = {
    "fp32_toy_cudacore": (CONFIGS["toy"], 0),
    "bf16_7b_tc": (scaled(CONFIGS["qwen7b"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 257, 416, 129 + 128],
                          budget=128, free_slack=5), 0),
    "bf16_7b_cudacore": (scaled(CONFIGS["qwen7b"], L=1, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 257], budget=128,
                                free_slack=5), zipc.ZPC_F_SCORE_CUDACORE),
    "bf16_8b_mixed_tc": (scaled(CONFIGS["llama8b"], L=2, h_kv=2, h_q=8, n_max=9, seq_lens=[513, 700, 1030],
                                budget=(32, 128), wave=0), 0),
    "bf16_32b_d64_tc": (scaled(CONFIGS["qwen32b"], L=2, h_kv=2, h_q=10, d=64, n_max=6, seq_lens=[200, 333],
                               budget=80, wave=0), 0),
    "bf16_prefix_tc": (scaled(CONFIGS["prefix"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[400] * 3,
                              prefix_tokens=160, budget=128, wave=0, free_slack=4), 0),
}


def _lse_input(w, inp, perturb_seed=None):
    """fp32 [L][M][w][h_q] normalisers from the oracle's definition (optionally perturbed)."""
    geo = geometry(w)
    lse = O.all_window_lse(geo, inp["q"], inp["k"], inp["slots"], inp["seq"], inp["tables"])
    if perturb_seed is not None:
        lse = lse + np.random.default_rng(perturb_seed).uniform(-0.5, 0.5, lse.shape)
    return lse.astype(np.float32)


def _run(cfg, seed, flags, perturb_seed=None, stages=False):
    w = from_host(make_host_workload(cfg, seed))
    inp = snapshot_inputs(w)
    lse32 = _lse_input(w, inp, perturb_seed)
    w.window_lse = torch.from_numpy(lse32).cuda()
    desc, params = desc_params(w, flags=flags, lse_input=True)
    b = batch_of(w, desc, params)
    if stages:
        for fn in (zipc.zpc_plan, zipc.zpc_score, zipc.zpc_select, zipc.zpc_compact, zipc.zpc_finalize):
            fn(desc, params, b)
    else:
        zipc.zpc_compress(desc, params, b)
    torch.cuda.synchronize()
    res = gpu_results(w, desc, params)
    full_check(w, inp, res, window_lse_in=lse32.astype(np.float64))
    return w, desc, params, lse32


@pytest.mark.parametrize("name", list(CASES))
def test_lse_input_parity(cuda_ok, name):
    cfg, flags = CASES[name]
    _run(cfg, 41, flags)


@pytest.mark.parametrize("name", ["bf16_7b_tc", "fp32_toy_cudacore", "bf16_8b_mixed_tc"])
def test_lse_input_is_used(cuda_ok, name):
    """Normalisers perturbed by U(-0.5, 0.5): the scores follow the given values (parity against the
    oracle fed the same perturbed array), so nothing recomputes them."""
    cfg, flags = CASES[name]
    _run(cfg, 42, flags, perturb_seed=9)


def test_lse_region_holds_the_input(cuda_ok):
    cfg, flags = CASES["bf16_7b_tc"]
    w, desc, params, lse32 = _run(cfg, 43, flags, stages=True)
    G = cfg.h_q // cfg.h_kv
    R = len(cfg.seq_lens)
    got = workspace_view(w, desc, params, "lse", torch.float32, (R, cfg.L, cfg.h_kv, cfg.w, G)).cpu().numpy()
    slots = w.q_slots.cpu().numpy()
    for r in range(R):
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                want = lse32[l, slots[r]][:, h * G:(h + 1) * G] * np.float32(1.4426950408889634)
                np.testing.assert_allclose(got[r, l, h], want, rtol=2e-7, atol=0)


def test_lse_input_requires_pointer(cuda_ok):
    cfg, _ = CASES["bf16_7b_tc"]
    w = from_host(make_host_workload(cfg, 44))
    desc, params = desc_params(w, lse_input=True)
    with pytest.raises(zipc.ZipcError):
        zipc.zpc_compress(desc, params, batch_of(w, desc, params))
