"""Full-size parity: BASELINE configs[1] (Qwen2.5-7B shape, 64 requests x 8192 tokens) in the
launch configuration bench.py times, checked against the oracle on sampled units (inputs for the
oracle are regenerated on the host by the numpy Philox generator, never read back from the GPU
generator) plus size-independent invariants on every unit and request."""
import math

import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params, workspace_view
from zpc_inputs import CONFIGS, budgets_for, k_rows, q_rows, v_rows
from zpc_inputs.device import generate

from helpers import check_band, check_band_tokens, check_scores, redundancy_eps

pytestmark = pytest.mark.gpu

SAMPLES = [(0, 0, 0), (37, 13, 2), (63, 27, 3), (5, 21, 1)]


@pytest.fixture(scope="module")
def run7b():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CONFIGS["qwen7b"]
    rids = np.arange(cfg.R)
    w = generate(cfg, 2603, rids)
    tables0 = w.layout.tables.copy()
    # pristine rows of the sampled units' target blocks are not needed: sources are regenerated
    desc, params = desc_params(w, flags=zipc.ZPC_F_COUNT_MOVES)
    b = batch_of(w, desc, params)
    zipc.zpc_compress(desc, params, b)
    torch.cuda.synchronize()
    return cfg, w, desc, params, tables0


def test_status_and_structure(run7b):
    cfg, w, desc, params, tables0 = run7b
    assert int(w.status.item()) == 0
    R = cfg.R
    T = 8192
    N = T // cfg.b
    nm = cfg.n_max
    new_lens = w.new_lens.cpu().numpy()
    np.testing.assert_array_equal(new_lens, np.minimum(T, w.budgets_host))
    tables = w.tables.cpu().numpy()
    # no prefix: in place: first N_max entries are the request's own first N_max blocks
    np.testing.assert_array_equal(tables[:, :nm], tables0[:, :nm])
    assert (w.new_num_blocks.cpu().numpy() == nm).all()
    freed = w.freed.cpu().numpy()[:int(w.num_freed.item())]
    expect = np.concatenate([tables0[r, nm:N] for r in range(R)])
    np.testing.assert_array_equal(freed, expect)
    top0 = w.layout.free_top
    assert int(w.free_top.item()) == top0 + len(expect)
    np.testing.assert_array_equal(w.free_stack.cpu().numpy()[top0:top0 + len(expect)], expect)


def test_kept_lists_all_units(run7b):
    """Every unit: kept list strictly ascending, length min(T, budget), window always kept."""
    cfg, w, desc, params, _ = run7b
    R = cfg.R
    lay = zipc.zpc_workspace_layout_get(desc, params, R)
    units = R * cfg.L * cfg.h_kv
    kept = workspace_view(w, desc, params, "kept", torch.int32, (units, lay.kept_stride))
    ell = w.new_lens.reshape(-1)
    T = 8192
    rng = torch.arange(lay.kept_stride, device=kept.device)
    valid = rng[None, :] < ell[:, None]
    k = torch.where(valid, kept, torch.full_like(kept, T))
    assert bool(((k[:, 1:] > k[:, :-1]) | ~valid[:, 1:]).all())
    assert bool(((k >= 0) & (k <= T)).all())
    # window tokens T-w..T-1 are the last w kept entries of every unit
    last = torch.gather(kept, 1, (ell[:, None] - cfg.w + torch.arange(cfg.w, device=kept.device)[None, :]).long())
    assert bool((last == torch.arange(T - cfg.w, T, device=kept.device)[None, :]).all())


def check_sampled_unit(cfg, w, desc, params, tables0, r, l, h, seed=2603):
    """One unit of a device-generated batch (global request id r = batch index r) against the oracle:
    scores, band rule, strict select, and the moved K/V bytes in the target blocks."""
    T = int(w.layout.seq_lens[r])
    # host regeneration of this unit's inputs (logical order), independent of the GPU generator
    kt = k_rows(cfg, seed, r, l, h, np.arange(T), T)                 # bf16 bits [T, d]
    q = q_rows(cfg, seed, r, l)                                       # [w, h_q, d]
    N = -(-T // cfg.b)
    kpad = np.zeros((N * cfg.b, cfg.d), kt.dtype)
    kpad[:T] = kt
    geo = O.Geometry(L=1, h_kv=1, h_q=cfg.G, d=cfg.d, b=cfg.b, N_total=N, M=1, w=cfg.w, dtype="bf16")
    kf = O.widen(kpad, "bf16").reshape(N, cfg.b, 1, cfg.d)
    qf = O.widen(q[:, h * cfg.G:(h + 1) * cfg.G, :], "bf16")
    s_ref = O.attention_scores(O.logits_dense(geo, qf, kf, np.arange(N), T, 0), T)
    R = len(w.layout.seq_lens)
    units = R * cfg.L * cfg.h_kv
    lay = zipc.zpc_workspace_layout_get(desc, params, R)
    u = (r * cfg.L + l) * cfg.h_kv + h
    S = workspace_view(w, desc, params, "scores", torch.float32, (units, w.max_seq_len))[u, :T].cpu().numpy()
    check_scores(S, s_ref, f"unit {r},{l},{h}")
    ell = int(w.new_lens[r, l, h].item())
    kept = workspace_view(w, desc, params, "kept", torch.int32, (units, lay.kept_stride))[u, :ell].cpu().numpy()
    check_band(kept, O.pin_window(O.max_pool(s_ref, cfg.pool_kernel), T, cfg.w), ell, f"unit {r},{l},{h}")
    sel = O.select(O.pin_window(O.max_pool(S.astype(np.float64), cfg.pool_kernel), T, cfg.w), ell)
    np.testing.assert_array_equal(sel, kept)
    # bytes: rank i of the unit now holds the original row kept[i] (K and V), in the target blocks
    vt = v_rows(cfg, seed, r, l, h, kept)
    tbl = tables0[r]
    ranks = np.arange(ell)
    blk = torch.from_numpy(tbl[ranks // cfg.b].astype(np.int64)).to(w.k.device)
    slot = torch.from_numpy((ranks % cfg.b).astype(np.int64)).to(w.k.device)
    k_now = w.k[l][blk, slot, h].cpu().numpy().view(np.uint16)
    v_now = w.v[l][blk, slot, h].cpu().numpy().view(np.uint16)
    np.testing.assert_array_equal(k_now, kt[kept])
    np.testing.assert_array_equal(v_now, vt)


@pytest.mark.parametrize("r,l,h", SAMPLES)
def test_sampled_units_vs_oracle(run7b, r, l, h):
    check_sampled_unit(*run7b, r, l, h)


# ---- NEXT-1 at full size: the bench's launch configuration with ZPC_F_REDUNDANCY
RED = (0.2, 0.4, 0.8)


@pytest.fixture(scope="module")
def run7b_red():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CONFIGS["qwen7b"]
    w = generate(cfg, 2603, np.arange(cfg.R))
    tables0 = w.layout.tables.copy()
    desc, params = desc_params(w, flags=zipc.ZPC_F_COUNT_MOVES, redundancy=RED)
    zipc.zpc_compress(desc, params, batch_of(w, desc, params))
    torch.cuda.synchronize()
    return cfg, w, desc, params, tables0


def test_redundancy_structure_full(run7b_red):
    cfg, w, desc, params, tables0 = run7b_red
    assert int(w.status.item()) == 0
    np.testing.assert_array_equal(w.new_lens.cpu().numpy(), np.minimum(8192, w.budgets_host))
    lay = zipc.zpc_workspace_layout_get(desc, params, cfg.R)
    units = cfg.R * cfg.L * cfg.h_kv
    kept = workspace_view(w, desc, params, "kept", torch.int32, (units, lay.kept_stride))
    ell = w.new_lens.reshape(-1)
    last = torch.gather(kept, 1, (ell[:, None] - cfg.w + torch.arange(cfg.w, device=kept.device)[None, :]).long())
    assert bool((last == torch.arange(8192 - cfg.w, 8192, device=kept.device)[None, :]).all())
    r = workspace_view(w, desc, params, "redundancy", torch.float32, (units, w.max_seq_len))[:, :8192]
    # each row sums at most b-1 cosines in [-1, 1], divided by T
    assert bool(torch.isfinite(r).all()) and bool((r.abs() <= (cfg.b - 1) / 8192 * (1 + 1e-5)).all())


@pytest.mark.parametrize("r,l,h", SAMPLES)
def test_redundancy_sampled_units_vs_oracle(run7b_red, r, l, h):
    cfg, w, desc, params, tables0 = run7b_red
    T, seed = 8192, 2603
    kt = k_rows(cfg, seed, r, l, h, np.arange(T), T)
    keys = O.widen(kt, "bf16").astype(np.float64)
    units = cfg.R * cfg.L * cfg.h_kv
    u = (r * cfg.L + l) * cfg.h_kv + h
    rr = workspace_view(w, desc, params, "redundancy", torch.float32, (units, w.max_seq_len))[u, :T].cpu().numpy()
    ref = O.lightning_redundancy_raw(keys, cfg.b, RED[2])
    # threshold decisions are discrete: compare the blocks whose cosines all keep 2e-5 from p
    ok = np.ones(T, bool)
    for j0 in range(0, T, cfg.b):
        C = O.cosine_matrix(keys[j0:j0 + cfg.b])
        if np.abs(C[~np.eye(cfg.b, dtype=bool)] - RED[2]).min() < 2e-5:
            ok[j0:j0 + cfg.b] = False
    assert ok.mean() > 0.9
    np.testing.assert_allclose(rr[ok], ref[ok], rtol=1e-5, atol=4e-5 / T)
    # kept band on the oracle's combined score (absolute band: S' may cross zero)
    q = q_rows(cfg, seed, r, l)
    geo = O.Geometry(L=1, h_kv=1, h_q=cfg.G, d=cfg.d, b=cfg.b, N_total=T // cfg.b, M=1, w=cfg.w, dtype="bf16")
    kf = O.widen(kt, "bf16").reshape(T // cfg.b, cfg.b, 1, cfg.d)
    qf = O.widen(q[:, h * cfg.G:(h + 1) * cfg.G, :], "bf16")
    pooled = O.max_pool(O.attention_scores(O.logits_dense(geo, qf, kf, np.arange(T // cfg.b), T, 0), T),
                        cfg.pool_kernel)
    s_ref = O.pin_window(O.combine_redundancy(pooled, ref, RED[0], RED[1]), T, cfg.w)
    lay = zipc.zpc_workspace_layout_get(desc, params, cfg.R)
    ell = int(w.new_lens[r, l, h].item())
    kg = workspace_view(w, desc, params, "kept", torch.int32, (units, lay.kept_stride))[u, :ell].cpu().numpy()
    # per-token band (tokens of ambiguous blocks get one cosine / T of slack in r)
    eps = redundancy_eps(pooled, ref, T, RED[0], RED[1], ambiguous=~ok)
    nk, nd = check_band_tokens(kg, s_ref, eps, ell, f"unit {r},{l},{h}")
    assert nk + nd >= 0.9 * T, (nk, nd)
    # strict: the GPU's own S and r through the oracle's combine + select, where the boundary is separated
    sg_raw = workspace_view(w, desc, params, "scores", torch.float32, (units, w.max_seq_len))[u, :T].cpu().numpy()
    sg = O.pin_window(O.combine_redundancy(O.max_pool(sg_raw.astype(np.float64), cfg.pool_kernel),
                                           rr.astype(np.float64), RED[0], RED[1]), T, cfg.w)
    vals = np.sort(sg)[::-1]
    gap = vals[ell - 1] - vals[ell]
    tight = 1e-6 * np.abs(pooled).max()          # the fp32 combine in k_select vs fp64 here
    if gap > tight:
        np.testing.assert_array_equal(O.select(sg, ell), kg)
    else:                                         # near-tie at the boundary (max pooling makes plateaus)
        check_band_tokens(kg, sg, np.full(T, tight), ell, f"unit {r},{l},{h} (own S')")


# ---- NEXT-4 at full size: single-pass scoring (ZPC_F_LSE_INPUT), the bench's --lse-input launch.
# The normalisers for all 7168 units come from the library's two-pass stage (standing in for the
# decode kernel); the sampled units are checked against the oracle's OWN exact normalisers, so an
# error in either pass fails.
@pytest.fixture(scope="module")
def run7b_lse():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from zpc_harness import window_lse_from_two_pass
    cfg = CONFIGS["qwen7b"]
    w = generate(cfg, 2603, np.arange(cfg.R))
    tables0 = w.layout.tables.copy()
    w.window_lse = window_lse_from_two_pass(w, zipc.ZPC_F_COUNT_MOVES)
    desc, params = desc_params(w, flags=zipc.ZPC_F_COUNT_MOVES, lse_input=True)
    zipc.zpc_compress(desc, params, batch_of(w, desc, params))
    torch.cuda.synchronize()
    return cfg, w, desc, params, tables0


def test_lse_input_structure_full(run7b_lse):
    test_status_and_structure(run7b_lse)
    test_kept_lists_all_units(run7b_lse)


@pytest.mark.parametrize("r,l,h", SAMPLES)
def test_lse_input_sampled_units_vs_oracle(run7b_lse, r, l, h):
    test_sampled_units_vs_oracle(run7b_lse, r, l, h)


# ---- NEXT-3: the paper's operating point at the bench's exact launch (4 requests x T = 2304,
# Qwen3-8B shape, b = 256, w = 16, N_max = 9; tcgen05 w = 16 path)
@pytest.fixture(scope="module")
def run_paper_op():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CONFIGS["paper_op"]
    w = generate(cfg, 2603, np.arange(cfg.wave))
    tables0 = w.layout.tables.copy()
    desc, params = desc_params(w, flags=zipc.ZPC_F_COUNT_MOVES)
    zipc.zpc_compress(desc, params, batch_of(w, desc, params))
    torch.cuda.synchronize()
    return cfg, w, desc, params, tables0


def test_paper_op_structure(run_paper_op):
    cfg, w, desc, params, tables0 = run_paper_op
    assert int(w.status.item()) == 0
    T, nm = 2304, cfg.n_max
    np.testing.assert_array_equal(w.new_lens.cpu().numpy(), np.minimum(T, w.budgets_host))
    tables = w.tables.cpu().numpy()
    np.testing.assert_array_equal(tables[:, :nm], tables0[:, :nm])
    assert int(w.num_freed.item()) == 0          # N = N_max: exactly one block's worth evicted, none freed
    R = cfg.wave
    units = R * cfg.L * cfg.h_kv
    lay = zipc.zpc_workspace_layout_get(desc, params, R)
    kept = workspace_view(w, desc, params, "kept", torch.int32, (units, lay.kept_stride))
    last = kept[:, 2048 - cfg.w:2048]
    assert bool((last == torch.arange(T - cfg.w, T, device=kept.device)[None, :]).all())


@pytest.mark.parametrize("r,l,h", [(0, 0, 0), (1, 17, 5), (3, 35, 7), (2, 8, 2)])
def test_paper_op_sampled_units_vs_oracle(run_paper_op, r, l, h):
    check_sampled_unit(*run_paper_op, r, l, h)
