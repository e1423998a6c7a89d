"""Pins of the NEXT-1 oracle (lightning redundancy + temperature softmax + combine), against what
the paper and the mathematics fix — not against the oracle's own formula:

* PAPER.md:616 defines the lightning score as the original score restricted to similarities
  between keys of the same block: the per-block oracle must equal the full-matrix (naive,
  PAPER.md:502) computation run on the block-diagonal-masked similarity matrix, and with one block
  the two are the naive score itself;
* SPEC.md:283 worked case: identical keys across blocks, orthogonal within blocks -> R uniform;
* closed form for a block of m identical keys (every off-diagonal cosine is 1): per column the
  newest other row is zeroed, so the row sums are (m-1, ..., m-1, m-2, 0) -- the newest token is the
  least redundant ("we prioritize retaining newer tokens");
* "exceeding the threshold" is strict (R21): a cosine of exactly 24/25 at p = 24/25 is kept;
* softmax with temperature: tau = 1 is the textbook softmax, constant input is uniform,
  tau -> 0 tends to the one-hot argmax; lambda = 0 leaves S unchanged.
"""
import numpy as np
import pytest

import oracle as O


def _block_mask(T, b):
    m = np.zeros((T, T), bool)
    for j0 in range(0, T, b):
        m[j0:j0 + b, j0:j0 + b] = True
    return m


@pytest.mark.parametrize("seed", range(25))
def test_lightning_equals_block_diagonal_naive(seed):
    rng = np.random.default_rng(seed)
    b = [4, 8, 16][seed % 3]
    T = int(rng.integers(b, 5 * b + 1))           # ragged last block
    d = int(rng.integers(2, 17))
    p = [0.3, 0.5, 0.8][seed % 3]
    keys = rng.standard_normal((T, d))
    # plant near-duplicates so the threshold rule bites
    for _ in range(T // 3):
        i, j = rng.integers(0, T, 2)
        keys[j] = keys[i] + 0.05 * rng.standard_normal(d)
    a = O.lightning_redundancy_raw(keys, b, p)
    ref = O.redundancy_raw_masked(keys, _block_mask(T, b), p)
    np.testing.assert_allclose(a, ref, rtol=0, atol=1e-12)


def test_single_block_is_the_naive_score():
    rng = np.random.default_rng(7)
    keys = rng.standard_normal((16, 8))
    keys[5] = keys[2] * 3.0
    np.testing.assert_allclose(O.lightning_redundancy_raw(keys, 16, 0.5),
                               O.redundancy_raw_masked(keys, np.ones((16, 16), bool), 0.5), atol=1e-14)


def test_spec_cross_block_identity_is_ignored():
    """identical keys across blocks, orthogonal within blocks -> lightning R uniform,
    while the naive (full-matrix) score is not."""
    b, nblk = 4, 3
    e = np.eye(b)
    keys = np.concatenate([e] * nblk)                 # block k is the identity rows again
    T = b * nblk
    r = O.lightning_redundancy_raw(keys, b, 0.5)
    np.testing.assert_array_equal(r, np.zeros(T))
    np.testing.assert_allclose(O.softmax_temperature(r, 0.4), np.full(T, 1.0 / T))
    naive = O.redundancy_raw_masked(keys, np.ones((T, T), bool), 0.5)
    assert naive.max() > 0


@pytest.mark.parametrize("m", [2, 3, 5, 16])
def test_identical_block_closed_form(m):
    keys = np.tile(np.array([[1.0, 2.0, -3.0]]), (m, 1))
    r = O.lightning_redundancy_raw(keys, m, 0.8) * m
    expect = np.full(m, m - 1.0)
    expect[m - 1] = 0.0
    if m >= 2:
        expect[m - 2] = m - 2.0 if m > 2 else 0.0
    # m = 2: column 0 zeroes row 1, column 1 zeroes row 0 -> both 0
    np.testing.assert_allclose(r, expect)


def test_threshold_is_strict():
    keys = np.array([[3.0, 4.0], [4.0, 3.0]])          # cosine 24/25 exactly
    p = 24.0 / 25.0
    np.testing.assert_allclose(O.lightning_redundancy_raw(keys, 2, p) * 2, [p, p])   # not above p
    np.testing.assert_array_equal(O.lightning_redundancy_raw(keys, 2, 0.95), [0.0, 0.0])


def test_zero_norm_key_has_cosine_zero():
    keys = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 0.0]])
    r = O.lightning_redundancy_raw(keys, 3, 0.5)
    # rows 1 and 2 identical: each column's only above-p entry is zeroed -> all zero
    np.testing.assert_array_equal(r, [0.0, 0.0, 0.0])
    r2 = O.lightning_redundancy_raw(keys, 3, 1.0)     # nothing exceeds 1: row sums of the cosines
    np.testing.assert_allclose(r2 * 3, [0.0, 1.0, 1.0])


def test_temperature_softmax_limits():
    x = np.array([0.3, -1.0, 2.5, 0.0])
    e = np.exp(x - x.max())
    np.testing.assert_allclose(O.softmax_temperature(x, 1.0), e / e.sum(), rtol=1e-15)
    np.testing.assert_allclose(O.softmax_temperature(np.full(5, 3.7), 0.4), np.full(5, 0.2))
    np.testing.assert_allclose(O.softmax_temperature(x, 1e-3), [0, 0, 1, 0], atol=1e-12)
    assert abs(O.softmax_temperature(x, 0.4).sum() - 1.0) < 1e-15


def test_combine_lambda_zero_and_mass():
    rng = np.random.default_rng(3)
    s = rng.random(40)
    r = rng.random(40)
    np.testing.assert_array_equal(O.combine_redundancy(s, r, 0.0, 0.4), s)
    d = s - O.combine_redundancy(s, r, 0.2, 0.4)
    assert abs(d.sum() - 0.2) < 1e-12 and (d > 0).all()


def test_compress_with_redundancy_follows_the_pipeline():
    """compress(F_REDUNDANCY) = attention score -> pool -> S - lambda softmax(r/tau) -> pin -> top-l."""
    from zpc_inputs import CONFIGS, make_host_workload, scaled
    cfg = scaled(CONFIGS["qwen7b"], L=1, h_kv=1, h_q=2, d=64, n_max=5, seq_lens=[90], budget=40, free_slack=3)
    hw = make_host_workload(cfg, 5)
    lay = hw.layout
    geo = O.Geometry(L=1, h_kv=1, h_q=2, d=64, b=cfg.b, N_total=lay.N_total, M=lay.M, w=cfg.w, dtype=cfg.dtype)
    prm = O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel, flags=O.F_REDUNDANCY, lam=0.2, tau=0.4, sim_p=0.8)
    out = O.compress(geo, prm, hw.k_cache, hw.v_cache, hw.q_cache, lay.q_slots, lay.seq_lens, lay.tables,
                     hw.budgets, None, lay.free_stack, lay.free_top)
    assert out.status == O.OK
    T = int(lay.seq_lens[0])
    kf = O.widen(hw.k_cache, cfg.dtype)
    s = out.scores[(0, 0, 0)]
    r = O.lightning_redundancy_raw(O.unit_keys(geo, kf, lay.tables[0], T, 0, 0), cfg.b, 0.8)
    np.testing.assert_array_equal(out.redundancy[(0, 0, 0)], r)
    manual = O.select(O.pin_window(O.max_pool(s, cfg.pool_kernel) - 0.2 * O.softmax_temperature(r, 0.4), T, cfg.w),
                      40)
    np.testing.assert_array_equal(out.kept[(0, 0, 0)], manual)
