"""GPU parity of NEXT-1 (ZPC_F_REDUNDANCY): lightning redundancy + temperature softmax folded into the
selection score, through the C ABI against the fp64 oracle.

Rules (NEXT-1):
* r[t] (row sums / T, the `redundancy` workspace region) within 4e-5/T absolute + 1e-5 relative of
  the oracle: fp32 cosines from exact bf16/fp32 inputs are within ~1e-6, and a row sums <= b-1 of
  them. The threshold decision "cos > p" is discrete: units whose oracle cosines come within 2e-5
  of p anywhere are skipped (both sides would be right), the rest must agree.
* kept sets: band rule on the oracle's combined score S' = pool(S) - lambda softmax(r / tau) with an
  absolute band of 1e-3 * max pool(S) (S' may cross zero, a relative band is meaningless there);
  and, where the l-th and (l+1)-th values of the GPU's own S' (recomputed in fp64 from the GPU's S and
  r) are separated, the oracle's selection on it must equal the GPU's kept list exactly.
* bytes: oracle compaction driven by the GPU's kept lists reproduces the whole pool bit-exactly.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params, workspace_view
from zpc_inputs import CONFIGS, make_host_workload, scaled
from zpc_inputs.device import from_host, to_host

from helpers import check_band_tokens, check_scores, redundancy_eps, geometry, gpu_results, snapshot_inputs, unit_index

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["select_auto", "select_reg", "red_mmasync"])
def _select_path(request, monkeypatch):
    """Run every case through both selection kernels: k_select (what these small T get by default)
    and the register-resident k_select_reg (params.variant select = 2 forces it for T <= 32K); and the
    b = 32..256 cases through both block-Gram kernels: k_red_umma (tcgen05, default) and k_red_tile
    (mma.sync, params.variant ZPC_V_RED_MMASYNC)."""
    monkeypatch.setattr(zipc, "DEFAULT_VARIANT", zipc.variant(select=2 if request.param == "select_reg" else 0,
                                                              red_mmasync=request.param == "red_mmasync"))

LAM, TAU, P = 0.2, 0.4, 0.8
MARGIN = 2e-5




def _run(cfg, seed, stages=False, p=P):
    hw = make_host_workload(cfg, seed)
    w = from_host(hw)
    inp = snapshot_inputs(w)
    desc, params = desc_params(w, redundancy=(LAM, TAU, p))
    b = batch_of(w, desc, params)
    if stages:
        for fn in (zipc.zpc_plan, zipc.zpc_score, zipc.zpc_redundancy, zipc.zpc_select, zipc.zpc_compact,
                   zipc.zpc_finalize):
            fn(desc, params, b)
    else:
        zipc.zpc_compress(desc, params, b)
    torch.cuda.synchronize()
    R = int(w.seq_lens.numel())
    units = R * cfg.L * cfg.h_kv
    res = gpu_results(w, desc, params)
    res["r"] = workspace_view(w, desc, params, "redundancy", torch.float32, (units, w.max_seq_len)).cpu().numpy()
    return w, inp, res


def _min_margin(keys, b, p):
    """min |cos - p| over the valid off-diagonal pairs of every block (fp64)."""
    T = keys.shape[0]
    best = np.inf
    for j0 in range(0, T, b):
        C = O.cosine_matrix(keys[j0:j0 + b])
        m = ~np.eye(C.shape[0], dtype=bool)
        if m.any():
            best = min(best, np.abs(C[m] - p).min())
    return best


CASES = {
    "fp32_toy_b4_generic": scaled(CONFIGS["toy"], pool_kernel=3),
    "bf16_7b_b16_mma": scaled(CONFIGS["qwen7b"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 257, 416, 129 + 128],
                              budget=128, free_slack=5),
    "bf16_32b_d64_mma": scaled(CONFIGS["qwen32b"], L=2, h_kv=2, h_q=10, d=64, n_max=6, seq_lens=[200, 333], budget=80,
                               wave=0),
    "bf16_b8_generic": scaled(CONFIGS["qwen7b"], L=1, h_kv=2, h_q=14, b=8, n_max=17, seq_lens=[300, 211], budget=128,
                              free_slack=5),
    # k_red_tile: b = 64 with a ragged last block, and the paper's operating point b = 256
    "bf16_b64_tile": scaled(CONFIGS["qwen7b"], L=1, h_kv=2, h_q=14, b=64, n_max=5, seq_lens=[300, 270], budget=200,
                            free_slack=5),
    "bf16_b256_tile": scaled(CONFIGS["paper_op"], L=2, h_kv=2, h_q=8, seq_lens=[2304, 2149], budget=2048, wave=0,
                             free_slack=4),
    # more blocks than SMs: every SM runs several k_red_umma CTAs over the call
    "bf16_b256_many": scaled(CONFIGS["paper_op"], L=4, h_kv=8, h_q=32, seq_lens=[2304, 2149, 2304, 2500], budget=2048,
                             wave=0, free_slack=6),
    "bf16_b48_d64_tile": scaled(CONFIGS["qwen32b"], L=1, h_kv=2, h_q=10, d=64, b=48, n_max=6, seq_lens=[250, 290],
                                budget=200, wave=0, free_slack=4),
}


@pytest.mark.parametrize("name", list(CASES))
def test_redundancy_rows_match_oracle(cuda_ok, name):
    cfg = CASES[name]
    w, inp, res = _run(cfg, seed=21)
    geo = geometry(w)
    kf = O.widen(inp["k"], cfg.dtype)
    checked = 0
    for r in range(len(inp["seq"])):
        T = int(inp["seq"][r])
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                keys = O.unit_keys(geo, kf, inp["tables"][r], T, l, h)
                if _min_margin(keys, cfg.b, P) < MARGIN:
                    continue
                ref = O.lightning_redundancy_raw(keys, cfg.b, P)
                got = res["r"][unit_index(w, r, l, h), :T]
                np.testing.assert_allclose(got, ref, rtol=1e-5, atol=4e-5 / T, err_msg=f"{name} r={r} l={l} h={h}")
                checked += 1
    assert checked >= max(1, (len(inp["seq"]) * cfg.L * cfg.h_kv) // 2), f"too many ambiguous units ({checked})"


P_LOW = 0.35   # ~4 standard deviations of a random 128-d cosine: a few dozen pairs per unit lie above it


@pytest.mark.parametrize("name", [n for n in CASES if "toy" not in n])
def test_redundancy_rows_zeroing_exercised(cuda_ok, name):
    """At p = 0.8 random keys never reach the threshold, so the "last row above p" zeroing
    would go untested; at p = 0.35 several cosines per unit exceed it (asserted), through every kernel."""
    cfg = CASES[name]
    w, inp, res = _run(cfg, seed=24, p=P_LOW)
    geo = geometry(w)
    kf = O.widen(inp["k"], cfg.dtype)
    checked = above = 0
    for r in range(len(inp["seq"])):
        T = int(inp["seq"][r])
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                keys = O.unit_keys(geo, kf, inp["tables"][r], T, l, h)
                if _min_margin(keys, cfg.b, P_LOW) < MARGIN:
                    continue
                for j0 in range(0, T, cfg.b):
                    C = O.cosine_matrix(keys[j0:j0 + cfg.b])
                    above += int((C[~np.eye(C.shape[0], dtype=bool)] > P_LOW).sum())
                ref = O.lightning_redundancy_raw(keys, cfg.b, P_LOW)
                got = res["r"][unit_index(w, r, l, h), :T]
                np.testing.assert_allclose(got, ref, rtol=1e-5, atol=4e-5 / T, err_msg=f"{name} r={r} l={l} h={h}")
                checked += 1
    assert checked >= max(1, (len(inp["seq"]) * cfg.L * cfg.h_kv) // 2), f"too many ambiguous units ({checked})"
    assert above > 0, "no cosine above p: the zeroing rule was not exercised"


@pytest.mark.parametrize("name,stages", [("fp32_toy_b4_generic", False), ("bf16_7b_b16_mma", False),
                                         ("bf16_7b_b16_mma", True), ("bf16_32b_d64_mma", False),
                                         ("bf16_b64_tile", False), ("bf16_b256_tile", False),
                                         ("bf16_b256_tile", True), ("bf16_b48_d64_tile", False)])
def test_redundancy_compress_parity(cuda_ok, name, stages):
    cfg = CASES[name]
    w, inp, res = _run(cfg, seed=22, stages=stages)
    geo = geometry(w)
    prm = O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel, max_seq_len=w.max_seq_len,
                   flags=O.F_REDUNDANCY | (O.F_PREFIX if w.layout.ref_counts is not None else 0),
                   lam=LAM, tau=TAU, sim_p=P)
    ref = O.compress(geo, prm, inp["k"], inp["v"], inp["q"], inp["slots"], inp["seq"], inp["tables"], inp["budgets"],
                     inp["refs"], inp["stack"], inp["top"], free_capacity=len(inp["stack"]),
                     freed_capacity=len(to_host(w.freed)))
    assert res["status"] == ref.status == O.OK
    kf = O.widen(inp["k"], cfg.dtype)
    gpu_kept = {}
    strict = decided = 0
    for r in range(len(inp["seq"])):
        T = int(inp["seq"][r])
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                key, u = (r, l, h), unit_index(w, r, l, h)
                where = f"{name} r={r} l={l} h={h}"
                check_scores(res["S"][u, :T], ref.scores[key], where)
                ell = int(res["new_lens"][r, l, h])
                assert ell == ref.new_lens[r, l, h], where
                kg = res["kept"][u, :ell].copy()
                gpu_kept[key] = kg
                assert np.all(np.diff(kg) > 0), where
                pooled = O.max_pool(ref.scores[key], cfg.pool_kernel)
                s_ref = O.pin_window(O.combine_redundancy(pooled, ref.redundancy[key], LAM, TAU), T, cfg.w)
                eps = redundancy_eps(pooled, ref.redundancy[key], T, LAM, TAU)
                band = 1e-3 * np.abs(pooled).max()
                nk, nd = check_band_tokens(kg, s_ref, eps, ell, where)
                decided += nk + nd
                kept = np.zeros(T, bool)
                kept[kg] = True
                assert np.all(kept[T - cfg.w:T]), f"{where}: window token dropped"
                # the GPU's own S and r through the oracle's combine + select (unambiguous boundary only)
                keys = O.unit_keys(geo, kf, inp["tables"][r], T, l, h)
                if _min_margin(keys, cfg.b, P) >= MARGIN:
                    sg = O.pin_window(O.combine_redundancy(O.max_pool(res["S"][u, :T].astype(np.float64),
                                                                      cfg.pool_kernel),
                                                           res["r"][u, :T].astype(np.float64), LAM, TAU), T, cfg.w)
                    vals = np.sort(sg)[::-1]
                    if ell < T and (not np.isfinite(vals[ell - 1]) or vals[ell - 1] - vals[ell] > 1e-6 * band / 1e-3):
                        np.testing.assert_array_equal(O.select(sg, ell), kg, err_msg=where)
                        strict += 1
    assert strict > 0
    # the per-token rule must decide almost every token (a vacuous band would decide few)
    assert decided >= 0.9 * sum(int(t) for t in inp["seq"]) * cfg.L * cfg.h_kv, decided
    ref2 = O.compress(geo, O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel, max_seq_len=w.max_seq_len,
                                    flags=prm.flags & ~O.F_REDUNDANCY), inp["k"], inp["v"], inp["q"], inp["slots"],
                      inp["seq"], inp["tables"], inp["budgets"], inp["refs"], inp["stack"], inp["top"],
                      kept_override=gpu_kept, free_capacity=len(inp["stack"]), freed_capacity=len(to_host(w.freed)))
    np.testing.assert_array_equal(res["k"], ref2.k_cache)
    np.testing.assert_array_equal(res["v"], ref2.v_cache)
    np.testing.assert_array_equal(res["tables"], ref2.fin.tables)
    np.testing.assert_array_equal(res["freed"], ref2.fin.freed)
    assert res["top"] == ref2.fin.free_top


def test_redundancy_flag_off_is_unchanged(cuda_ok):
    """Without the flag the redundancy stage is a no-op and the kept lists are the plain method's."""
    cfg = CASES["bf16_7b_b16_mma"]
    hw = make_host_workload(cfg, 23)
    outs = []
    for red in (None, (0.0, TAU, P)):      # lambda = 0: S - 0*R == S
        w = from_host(hw)
        desc, params = desc_params(w, redundancy=red)
        zipc.zpc_compress(desc, params, batch_of(w, desc, params))
        torch.cuda.synchronize()
        outs.append((to_host(w.new_lens), to_host(w.k, True), to_host(w.tables)))
    for a, b in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, b)

