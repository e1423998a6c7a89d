"""Pins of the NEXT-2 oracle (global score, Alg. 2, and F relocation PAPER.md:595)
against hand-worked cases and identities the paper fixes:

* an uncompressed request only stores S (lines 3-4): F <- S, selection unchanged;
* alpha = 0 leaves S unchanged for a compressed request (max(0*f, s) = s, scores are >= 0);
* a hand-worked Alg. 2 instance: T = 10, b = 4, N_max = 3 -> blocks 0, 1 take max(alpha f, s),
  block 2 (the last, no history, R25) keeps s; F holds the result;
* history that dominates gives S' = alpha * F on the history blocks;
* relocation: after compaction F at target rank i of head h equals the updated score of kept[i].
"""
import numpy as np

import oracle as O
from zpc_inputs import CONFIGS, make_host_workload, scaled


def test_alg2_hand_example():
    b, n_max, T, alpha = 4, 3, 10, 0.5
    table = [2, 0, 3]
    f = np.zeros((4, b, 1), np.float32)
    f[2, :, 0] = [0.8, 0.0, 0.2, 0.3]       # history of block 0 (physical 2)
    f[0, :, 0] = [0.1, 0.6, 0.0, 0.0]       # block 1 (physical 0)
    f[3, :, 0] = [9.0, 9.0, 9.0, 9.0]       # block 2 (physical 3): the last block, no history
    s = np.array([0.1, 0.2, 0.3, 0.05, 0.1, 0.1, 0.1, 0.1, 0.02, 0.03])
    out = O.global_score_update(s, f, table, T, 0, b, n_max, True, alpha)
    expect = s.copy()
    expect[0:4] = np.maximum(alpha * np.array([0.8, 0.0, 0.2, 0.3]), s[0:4])    # [0.4, 0.2, 0.3, 0.15]
    expect[4:8] = np.maximum(alpha * np.array([0.1, 0.6, 0.0, 0.0]), s[4:8])    # [0.1, 0.3, 0.1, 0.1]
    np.testing.assert_allclose(out, expect)
    np.testing.assert_allclose(out[:4], [0.4, 0.2, 0.3, 0.15])
    np.testing.assert_allclose(f[2, :, 0], np.float32(expect[0:4]))
    np.testing.assert_allclose(f[0, :, 0], np.float32(expect[4:8]))
    np.testing.assert_allclose(f[3, :2, 0], np.float32(s[8:10]))      # stored, not maxed
    np.testing.assert_array_equal(f[3, 2:, 0], [9.0, 9.0])             # slots >= T untouched


def test_shared_prefix_blocks_are_read_not_written():
    """R31: with n_prefix = 1 the first block (shared by several requests)
    still contributes alpha * F to the scores but its F entries are not overwritten; the private blocks
    are updated as in the hand example above."""
    b, n_max, T, alpha = 4, 3, 10, 0.5
    table = [2, 0, 3]
    f = np.zeros((4, b, 1), np.float32)
    f[2, :, 0] = [0.8, 0.0, 0.2, 0.3]
    f[0, :, 0] = [0.1, 0.6, 0.0, 0.0]
    s = np.array([0.1, 0.2, 0.3, 0.05, 0.1, 0.1, 0.1, 0.1, 0.02, 0.03])
    out = O.global_score_update(s, f, table, T, 0, b, n_max, True, alpha, n_prefix=1)
    np.testing.assert_allclose(out[:4], [0.4, 0.2, 0.3, 0.15])        # history still read
    np.testing.assert_array_equal(f[2, :, 0], np.float32([0.8, 0.0, 0.2, 0.3]))   # shared: unchanged
    np.testing.assert_allclose(f[0, :, 0], np.float32([0.1, 0.3, 0.1, 0.1]))      # private: updated
    f2 = np.zeros((4, b, 1), np.float32)
    out2 = O.global_score_update(s, f2, table, T, 0, b, n_max, False, alpha, n_prefix=2)
    np.testing.assert_array_equal(out2, s)                            # never compressed: S unchanged
    np.testing.assert_array_equal(f2[2], 0)
    np.testing.assert_array_equal(f2[0], 0)
    np.testing.assert_allclose(f2[3, :2, 0], np.float32(s[8:10]))


def test_uncompressed_stores_only():
    b, T = 4, 9
    f = np.full((3, b, 2), 7.0, np.float32)
    s = np.linspace(0.01, 0.2, T)
    out = O.global_score_update(s, f, [1, 2, 0], T, 1, b, 3, False, 0.8)
    np.testing.assert_array_equal(out, s)
    np.testing.assert_allclose(f[[1, 1, 1, 1, 2, 2, 2, 2, 0], [0, 1, 2, 3, 0, 1, 2, 3, 0], 1], np.float32(s))
    np.testing.assert_array_equal(f[:, :, 0], 7.0)                      # other head untouched


def _setup(seed=4, alpha=0.8, compressed=(1, 0)):
    cfg = scaled(CONFIGS["qwen7b"], L=1, h_kv=2, h_q=4, d=64, n_max=5, seq_lens=[90, 70], budget=40, free_slack=4)
    hw = make_host_workload(cfg, seed)
    lay = hw.layout
    geo = O.Geometry(L=1, h_kv=2, h_q=4, d=64, b=cfg.b, N_total=lay.N_total, M=lay.M, w=cfg.w, dtype=cfg.dtype)
    rng = np.random.default_rng(seed)
    f0 = (rng.random((1, lay.N_total, cfg.b, 2)) * 0.05).astype(np.float32)
    prm = O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel, flags=O.F_GLOBAL_SCORE, alpha=alpha)
    run = lambda p, f: O.compress(geo, p, hw.k_cache, hw.v_cache, hw.q_cache, lay.q_slots, lay.seq_lens,  # noqa: E731
                                  lay.tables, hw.budgets, None, lay.free_stack, lay.free_top, f_cache=f,
                                  is_compressed=np.array(compressed))
    return cfg, hw, geo, f0, prm, run


def test_uncompressed_request_selects_like_plain_method():
    cfg, hw, geo, f0, prm, run = _setup(compressed=(0, 0))
    g = run(prm, f0)
    plain = run(O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel), None)
    for key in plain.kept:
        np.testing.assert_array_equal(g.kept[key], plain.kept[key])
        np.testing.assert_array_equal(g.global_scores[key], g.scores[key])


def test_alpha_zero_is_identity_on_scores():
    cfg, hw, geo, f0, prm, run = _setup(alpha=0.0, compressed=(1, 1))
    g = run(prm, f0)
    for key in g.scores:
        np.testing.assert_array_equal(g.global_scores[key], g.scores[key])


def test_dominating_history_and_relocation():
    cfg, hw, geo, f0, prm, run = _setup(compressed=(1, 0))
    f_big = np.ones_like(f0)
    g = run(prm, f_big)
    lay = hw.layout
    hist = (cfg.n_max - 1) * cfg.b
    for (r, l, h), s in g.global_scores.items():
        T = int(lay.seq_lens[r])
        if r == 0:
            np.testing.assert_allclose(s[:min(T, hist)], 0.8)       # alpha * F dominates every score
            np.testing.assert_array_equal(s[hist:T], g.scores[(r, l, h)][hist:T])
        else:
            np.testing.assert_array_equal(s, g.scores[(r, l, h)])
        # relocation: F at target rank i = the updated score of kept[i] (fp32)
        kept = g.kept[(r, l, h)]
        tg = g.plan.targets[r]
        rank = np.arange(len(kept))
        np.testing.assert_array_equal(g.f_cache[l, np.asarray(tg)[rank // cfg.b], rank % cfg.b, h],
                                      np.float32(s[kept]))


def test_pool_first_only_pools_first_compressions():
    """R32: with F_POOL_FIRST a request compressed before (r = 0) selects on the unpooled
    score and a first-time request (r = 1) on the pooled one: each kept set equals the plain method's with
    that pool width, and the two widths really select differently here."""
    cfg, hw, geo, f0, prm, run = _setup(compressed=(1, 0))
    pf = run(O.Params(n_max=cfg.n_max, pool_kernel=7, flags=O.F_POOL_FIRST), None)
    pooled = run(O.Params(n_max=cfg.n_max, pool_kernel=7), None)
    unpooled = run(O.Params(n_max=cfg.n_max, pool_kernel=1), None)
    differ = False
    for (r, l, h), kept in pf.kept.items():
        ref = (unpooled if r == 0 else pooled).kept[(r, l, h)]
        np.testing.assert_array_equal(kept, ref)
        differ |= not np.array_equal(pooled.kept[(r, l, h)], unpooled.kept[(r, l, h)])
    assert differ
