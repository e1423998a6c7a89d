"""Pins of the NEXT-4 oracle functions (single-pass scoring with the window normalisers given):
window_lse, attention_scores_given_lse, unit_window_lse, all_window_lse, compress(window_lse_in=...).

What fixes each expected value: scipy's logsumexp (a library routine, not the oracle's formula), a
hand-worked example, the constant-keys closed form, exact scaling identities, and the
cross-check against attention_scores, which is pinned independently in test_oracle_pins.py.
"""
import math

import numpy as np
import pytest
from scipy.special import logsumexp

import oracle as O
from zpc_inputs import CONFIGS, make_host_workload, scaled


def _case(rng, G, w, d, b, T, h_kv=1):
    geo = O.Geometry(L=1, h_kv=h_kv, h_q=G * h_kv, d=d, b=b, N_total=-(-T // b) + 3, M=1, w=w, dtype="fp32")
    table = rng.permutation(geo.N_total)[:-(-T // b)]
    q = rng.standard_normal((w, geo.h_q, d))
    k = rng.standard_normal((geo.N_total, b, h_kv, d))
    return geo, q, k, table


def test_window_lse_is_scipy_logsumexp_over_the_causal_range():
    """LSE[g,u] = logsumexp of q_{g,u}.k_t/sqrt(d) over t <= T-w+u (scipy.special.logsumexp on the
    gathered keys)."""
    rng = np.random.default_rng(7)
    G, w, d, b, T = 3, 4, 8, 4, 19
    geo, q, k, table = _case(rng, G, w, d, b, T)
    lse = O.window_lse(O.logits_blockwise(geo, q, k, table, T, 0), T)
    Kd = np.stack([k[table[t // b], t % b, 0] for t in range(T)])
    for g in range(G):
        for u in range(w):
            x = Kd[:T - w + u + 1] @ q[u, g] / math.sqrt(d)
            assert abs(lse[g, u] - logsumexp(x)) < 1e-12


def test_hand_worked_lse_and_scores():
    """d=2, b=2, T=3, w=1, G=1: q=(1,2), keys (1,0),(0,1),(1,1) -> logits (1,2,3)/sqrt(2);
    LSE = log(e^{1/r2} + e^{2/r2} + e^{3/r2}); with LSE + 0.5 given, s[t] = e^{x_t - LSE - 0.5}."""
    geo = O.Geometry(L=1, h_kv=1, h_q=1, d=2, b=2, N_total=3, M=1, w=1, dtype="fp32")
    q = np.array([[[1.0, 2.0]]])
    k = np.zeros((3, 2, 1, 2))
    table = [2, 0]
    k[2, 0, 0] = [1, 0]; k[2, 1, 0] = [0, 1]; k[0, 0, 0] = [1, 1]
    A = O.logits_blockwise(geo, q, k, table, 3, 0)
    x = [1 / math.sqrt(2), 2 / math.sqrt(2), 3 / math.sqrt(2)]
    L = math.log(sum(math.exp(v) for v in x))
    assert abs(O.window_lse(A, 3)[0, 0] - L) < 1e-14
    s = O.attention_scores_given_lse(A, np.array([[L + 0.5]]), 3)
    np.testing.assert_allclose(s, [math.exp(v - L - 0.5) for v in x], rtol=1e-14)


@pytest.mark.parametrize("G,w,b,T", [(1, 3, 4, 10), (2, 4, 4, 13)])
def test_constant_keys_lse_closed_form(G, w, b, T):
    """All K rows equal: A[g,u,t] = c_{g,u} on t <= T-w+u, so LSE[g,u] = c_{g,u} + log(T-w+u+1)."""
    rng = np.random.default_rng(3)
    geo, q, k, table = _case(rng, G, w, 6, b, T)
    k[:] = k[0, 0]
    A = O.logits_dense(geo, q, k, table, T, 0)
    lse = O.window_lse(A, T)
    for g in range(G):
        for u in range(w):
            c = q[u, g] @ k[0, 0, 0] / math.sqrt(6)
            assert abs(lse[g, u] - (c + math.log(T - w + u + 1))) < 1e-12


@pytest.mark.parametrize("G,w", [(1, 1), (2, 3), (4, 2)])
def test_given_exact_lse_equals_two_pass_scores(G, w):
    """With the exact normalisers, the single-pass formula is the softmax of PAPER.md:409-411, i.e.
    attention_scores (pinned independently by closed forms and scipy softmax)."""
    rng = np.random.default_rng(11 + G)
    T = 23
    geo, q, k, table = _case(rng, G, w, 8, 4, T)
    A = O.logits_dense(geo, q, k, table, T, 0)
    np.testing.assert_allclose(O.attention_scores_given_lse(A, O.window_lse(A, T), T),
                               O.attention_scores(A, T), rtol=1e-12)


def test_uniform_shift_scales_scores():
    """Adding delta to every normaliser divides every score by e^delta (max and mean commute with a
    common positive factor)."""
    rng = np.random.default_rng(5)
    T = 17
    geo, q, k, table = _case(rng, 3, 2, 8, 4, T)
    A = O.logits_dense(geo, q, k, table, T, 0)
    lse = O.window_lse(A, T)
    np.testing.assert_allclose(O.attention_scores_given_lse(A, lse + 0.7, T),
                               O.attention_scores(A, T) * math.exp(-0.7), rtol=1e-12)


def test_per_head_shift_moves_the_gqa_max():
    """G=2, w=1, T=1 by hand: one key, logits a0, a1; with normalisers (a0, a1 + 2) the scores are
    max(e^0, e^-2) = 1; with (a0 + 3, a1) they are max(e^-3, e^0) = 1; with (a0+1, a1+2): e^-1."""
    A = np.array([[[0.25]], [[-1.5]]])          # [G=2, w=1, T=1]
    for lse, want in (([0.25, 0.5], 1.0), ([3.25, -1.5], 1.0), ([1.25, 0.5], math.exp(-1))):
        s = O.attention_scores_given_lse(A, np.array(lse)[:, None], 1)
        assert abs(s[0] - want) < 1e-15


def test_unit_window_lse_layout():
    """[L][M][w][h_q] indexing: entry (l, j, u, i) is picked for KV head h = i // G, column (g, u)."""
    geo = O.Geometry(L=2, h_kv=2, h_q=6, d=8, b=4, N_total=8, M=3, w=2, dtype="fp32")
    arr = np.zeros((2, 3, 2, 6))
    for l in range(2):
        for j in range(3):
            for u in range(2):
                for i in range(6):
                    arr[l, j, u, i] = 1000 * l + 100 * j + 10 * u + i
    x = O.unit_window_lse(geo, arr, slot=2, l=1, h=1)    # heads 3, 4, 5
    assert x.shape == (3, 2)
    for g in range(3):
        for u in range(2):
            assert x[g, u] == 1000 + 200 + 10 * u + (3 + g)


def test_compress_with_exact_lse_input_equals_two_pass():
    """compress(window_lse_in = all_window_lse(...)) reproduces the two-pass oracle: scores within
    1e-12, identical kept sets, pools and bookkeeping (toy and a GQA shape with ragged lengths)."""
    for cfg in (CONFIGS["toy"], scaled(CONFIGS["qwen7b"], L=1, h_kv=2, h_q=4, d=64, n_max=5, seq_lens=[70, 65],
                                        budget=40, free_slack=3, dtype="fp32")):
        hw = make_host_workload(cfg, seed=4)
        lay = hw.layout
        geo = O.Geometry(L=cfg.L, h_kv=cfg.h_kv, h_q=cfg.h_q, d=cfg.d, b=cfg.b, N_total=lay.N_total, M=lay.M,
                         w=cfg.w, dtype=cfg.dtype)
        prm = O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel)
        args = (geo, prm, hw.k_cache, hw.v_cache, hw.q_cache, lay.q_slots, lay.seq_lens, lay.tables, hw.budgets,
                None, lay.free_stack, lay.free_top)
        lse = O.all_window_lse(geo, hw.q_cache, hw.k_cache, lay.q_slots, lay.seq_lens, lay.tables)
        a, b = O.compress(*args), O.compress(*args, window_lse_in=lse)
        for key in a.scores:
            np.testing.assert_allclose(b.scores[key], a.scores[key], rtol=1e-12)
            np.testing.assert_array_equal(b.kept[key], a.kept[key])
        np.testing.assert_array_equal(b.k_cache, a.k_cache)
        np.testing.assert_array_equal(b.fin.freed, a.fin.freed)
