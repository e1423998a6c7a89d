"""Shared test glue: run the CUDA path through the C ABI and compare with the oracle (§8(c) rules)."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params, workspace_view
from zpc_inputs.device import to_host

SCORE_RTOL = 1e-3        # north_star: window scores within 1e-3 relative (fp32 accumulate from bf16)
SCORE_ATOL = 1e-30
BAND = 1e-3


def geometry(w):
    cfg, lay = w.cfg, w.layout
    return O.Geometry(L=cfg.L, h_kv=cfg.h_kv, h_q=cfg.h_q, d=cfg.d, b=cfg.b, N_total=lay.N_total, M=lay.M,
                      w=cfg.w, dtype=cfg.dtype)


def oparams(w, flags=0, pool=None):
    cfg = w.cfg
    f = flags | (O.F_PREFIX if w.layout.ref_counts is not None else 0)
    return O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel if pool is None else pool,
                    max_seq_len=w.max_seq_len, flags=f)


def snapshot_inputs(w):
    """Host copies of everything the call reads (taken BEFORE the call)."""
    u16 = w.cfg.dtype == "bf16"
    return dict(k=to_host(w.k, u16), v=to_host(w.v, u16), q=to_host(w.q, u16), tables=to_host(w.tables),
                seq=to_host(w.seq_lens), slots=to_host(w.q_slots), budgets=to_host(w.budgets),
                refs=None if w.ref_counts is None else to_host(w.ref_counts),
                stack=to_host(w.free_stack), top=int(w.free_top.item()))


def run_gpu(w, flags=0, pool=None, stages=False):
    desc, params = desc_params(w, flags=flags, pool_kernel=pool)
    b = batch_of(w, desc, params)
    if stages:
        for fn in (zipc.zpc_plan, zipc.zpc_score, zipc.zpc_select, zipc.zpc_compact, zipc.zpc_finalize):
            fn(desc, params, b)
    else:
        zipc.zpc_compress(desc, params, b)
    torch.cuda.synchronize()
    return desc, params


def gpu_results(w, desc, params):
    cfg = w.cfg
    R = int(w.seq_lens.numel())
    units = R * cfg.L * cfg.h_kv
    lay = zipc.zpc_workspace_layout_get(desc, params, R)
    S = workspace_view(w, desc, params, "scores", torch.float32, (units, w.max_seq_len)).cpu().numpy()
    kept = workspace_view(w, desc, params, "kept", torch.int32, (units, lay.kept_stride)).cpu().numpy()
    u16 = cfg.dtype == "bf16"
    return dict(status=int(w.status.item()), S=S, kept=kept, k=to_host(w.k, u16), v=to_host(w.v, u16),
                tables=to_host(w.tables), new_lens=to_host(w.new_lens), nnb=to_host(w.new_num_blocks),
                freed=to_host(w.freed)[:int(w.num_freed.item())], stack=to_host(w.free_stack),
                top=int(w.free_top.item()), refs=None if w.ref_counts is None else to_host(w.ref_counts))


def unit_index(w, r, l, h):
    return (r * w.cfg.L + l) * w.cfg.h_kv + h


def check_scores(s_gpu, s_ref, where=""):
    err = np.abs(s_gpu - s_ref)
    bad = err > SCORE_RTOL * np.abs(s_ref) + SCORE_ATOL
    assert not bad.any(), f"{where}: {bad.sum()} scores outside 1e-3 rel; worst at {np.argmax(err / (np.abs(s_ref) + 1e-300))}"


def check_band(kept_gpu, s_ref_final, ell, where=""):
    """Kept-set rule of §8(c): above theta(1+1e-3) must be kept, below theta(1-1e-3) dropped."""
    assert len(kept_gpu) == ell, where
    assert np.all(np.diff(kept_gpu) > 0), f"{where}: kept list not strictly ascending"
    order = np.sort(s_ref_final)[::-1]
    theta = order[ell - 1]
    kept = np.zeros(len(s_ref_final), bool)
    kept[kept_gpu] = True
    if np.isinf(theta):
        must = np.isinf(s_ref_final)
        assert np.all(kept[must]) or must.sum() > ell, where
        return
    must_keep = s_ref_final > theta * (1 + BAND)
    must_drop = s_ref_final < theta * (1 - BAND)
    assert np.all(kept[must_keep]), f"{where}: dropped a token above the band"
    assert not np.any(kept[must_drop]), f"{where}: kept a token below the band"


def check_band_tokens(kept_gpu, s_ref_final, eps, ell, where=""):
    """Kept-set rule with a per-token error allowance eps[t] >= |s_gpu[t] - s_ref[t]| (NEXT-1, where
    the combined score S' = pool(S) - lambda softmax(r / tau) may cross zero, so no relative band fits).
    With L = s_ref - eps and U = s_ref + eps: a token that fewer than ell others can possibly beat
    (#{j != t: U_j >= L_t} < ell) must be kept; one that at least ell others surely beat
    (#{j: L_j > U_t} >= ell) must be dropped. Returns (#must-keep, #must-drop) for coverage checks."""
    assert len(kept_gpu) == ell, where
    assert np.all(np.diff(kept_gpu) > 0), f"{where}: kept list not strictly ascending"
    s = np.asarray(s_ref_final, np.float64)
    fin = np.isfinite(s)
    lo = np.where(fin, s - eps, s)
    hi = np.where(fin, s + eps, s)
    hs, ls = np.sort(hi), np.sort(lo)
    n = len(s)
    beat_possible = n - np.searchsorted(hs, lo, side="left") - 1   # j != t with U_j >= L_t (U_t >= L_t)
    beat_sure = n - np.searchsorted(ls, hi, side="right")           # j with L_j > U_t
    must_keep = beat_possible < ell
    must_drop = beat_sure >= ell
    kept = np.zeros(n, bool)
    kept[kept_gpu] = True
    assert np.all(kept[must_keep]), f"{where}: dropped a token no error allowance could push out"
    assert not np.any(kept[must_drop]), f"{where}: kept a token at least ell others surely beat"
    return int(must_keep.sum()), int(must_drop.sum())


def redundancy_eps(pooled, r_ref, T, lam, tau, ambiguous=None):
    """Per-token allowance for |S'_gpu - S'_ref|, S' = pool(S) - lambda softmax(r / tau) (NEXT-1, R22):
    1e-3 pool(S)_t (the score tolerance; max pooling keeps it) + lambda |d softmax_t|. An error
    dr_j <= 1e-5 |r_j| + 4e-5 / T in r (the r tolerance of the NEXT-1 tests) moves softmax_t = e^{r_t/tau} / Z
    by at most softmax_t (e^{(dr_t + max_j dr_j) / tau} - 1). `ambiguous` marks tokens whose block has a
    cosine within the test margin of p: there the discrete zeroing may flip, moving r_t by one cosine
    (<= 1) / T."""
    dr = 1e-5 * np.abs(r_ref) + 4e-5 / T
    if ambiguous is not None:
        dr = np.where(ambiguous, dr + 1.0 / T, dr)
    sm = O.softmax_temperature(r_ref, tau)
    return 1e-3 * np.abs(pooled) + lam * sm * np.expm1((dr + dr.max()) / tau) + 1e-12


def full_check(w, inp, res, pool=None, strict_select=True, blockwise=False, window_lse_in=None,
               pool_first_compressed=None):
    """Every parity rule of §8(c) on a fully materialised (small) workload. window_lse_in: the
    normalisers given to a ZPC_F_LSE_INPUT call (NEXT-4), passed to the oracle as well.
    pool_first_compressed: the is_compressed[R] of a ZPC_F_POOL_FIRST call (R32): those requests select
    on the unpooled score."""
    pf = pool_first_compressed
    geo, prm = geometry(w), oparams(w, pool=pool, flags=O.F_POOL_FIRST if pf is not None else 0)
    cfg = w.cfg
    R = len(inp["seq"])
    ref = O.compress(geo, prm, inp["k"], inp["v"], inp["q"], inp["slots"], inp["seq"], inp["tables"],
                     inp["budgets"], inp["refs"], inp["stack"], inp["top"], blockwise=blockwise,
                     free_capacity=len(inp["stack"]), freed_capacity=len(to_host(w.freed)),
                     window_lse_in=window_lse_in, is_compressed=pf)
    assert res["status"] == ref.status == O.OK, (res["status"], ref.status)
    gpu_kept = {}
    for r in range(R):
        T = int(inp["seq"][r])
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                u = unit_index(w, r, l, h)
                key = (r, l, h)
                where = f"unit r={r} l={l} h={h}"
                check_scores(res["S"][u, :T], ref.scores[key], where)
                ell = int(res["new_lens"][r, l, h])
                assert ell == ref.new_lens[r, l, h], where
                kg = res["kept"][u, :ell].copy()
                gpu_kept[key] = kg
                kp = 1 if (pf is not None and pf[r]) else prm.pool_kernel
                s_final = O.pin_window(O.max_pool(ref.scores[key], kp), T, cfg.w)
                check_band(kg, s_final, ell, where)
                if strict_select:
                    # GPU's own fp32 S through the oracle's pool+pin+select: must match bit for bit
                    s32 = res["S"][u, :T].astype(np.float64)
                    sel = O.select(O.pin_window(O.max_pool(s32, kp), T, cfg.w), ell)
                    np.testing.assert_array_equal(sel, kg, err_msg=where)
    # bytes: oracle compaction driven by the GPU's kept lists reproduces the whole pool
    ref2 = O.compress(geo, prm, inp["k"], inp["v"], inp["q"], inp["slots"], inp["seq"], inp["tables"],
                      inp["budgets"], inp["refs"], inp["stack"], inp["top"], kept_override=gpu_kept,
                      free_capacity=len(inp["stack"]), freed_capacity=len(to_host(w.freed)), is_compressed=pf)
    np.testing.assert_array_equal(res["k"], ref2.k_cache)
    np.testing.assert_array_equal(res["v"], ref2.v_cache)
    np.testing.assert_array_equal(res["tables"], ref2.fin.tables)
    np.testing.assert_array_equal(res["nnb"], ref2.fin.new_num_blocks)
    np.testing.assert_array_equal(res["freed"], ref2.fin.freed)
    assert res["top"] == ref2.fin.free_top
    np.testing.assert_array_equal(res["stack"][:res["top"]], ref2.fin.free_stack[:ref2.fin.free_top])
    if res["refs"] is not None:
        np.testing.assert_array_equal(res["refs"], ref2.fin.ref_counts)
    return ref
