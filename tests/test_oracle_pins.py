"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test cites what fixes the expected value: the paper's Fig. 1 structure,
closed forms, textbook routines (scipy softmax), brute force, or SPEC examples
restated for this ABI. Every stage has at least one pin that a plausible slip
(dropped term, wrong sign/index, transposed operand, max/mean order) would fail.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy.special import softmax as sp_softmax

import oracle as O
from zpc_inputs import CONFIGS, make_host_workload, scaled
from zpc_inputs.philox import philox4x32

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def geo_of(cfg, lay):
    return O.Geometry(L=cfg.L, h_kv=cfg.h_kv, h_q=cfg.h_q, d=cfg.d, b=cfg.b, N_total=lay.N_total,
                      M=lay.M, w=cfg.w, dtype=cfg.dtype)


# ------------------------------------------------------------------ generator
def test_philox_known_answers():
    """Random123 known-answer vectors for Philox4x32-10 (tests/golden/philox_kat.json)."""
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for case in kat["cases"]:
        c = [np.uint32(int(x, 16)) for x in case["ctr"]]
        k = [int(x, 16) for x in case["key"]]
        out = philox4x32(*c, *k)
        assert [f"{int(x):08x}" for x in out] == case["out"]


# ------------------------------------------------------------------ Fig. 1
def _toy(pool=1):
    cfg = scaled(CONFIGS["toy"], pool_kernel=pool)
    hw = make_host_workload(cfg, seed=1)
    lay = hw.layout
    geo = geo_of(cfg, lay)
    prm = O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel)
    out = O.compress(geo, prm, hw.k_cache, hw.v_cache, hw.q_cache, lay.q_slots, lay.seq_lens,
                     lay.tables, hw.budgets, None, lay.free_stack, lay.free_top)
    return cfg, hw, geo, out


@pytest.mark.parametrize("pool", [1, 3])
def test_fig1_toy_structure(pool):
    """PAPER.md:22 (Fig. 1 caption): N_max=4, b=4, w=2, two requests: kept entries go to
    the first three blocks, the fourth is reserved, the rest are released."""
    cfg, hw, geo, out = _toy(pool)
    lay = hw.layout
    assert out.status == O.OK
    A, B = lay.tables[0], lay.tables[1]
    assert list(out.fin.freed) == [A[4], B[4], B[5], B[6]]
    for r, T in enumerate([20, 25]):
        assert list(out.fin.tables[r, :4]) == list(lay.tables[r, :4])  # in place, same blocks
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                kept = out.kept[(r, l, h)]
                assert len(kept) == 12 == (cfg.n_max - 1) * cfg.b    # k = (N_max-1)*b
                assert {T - 2, T - 1} <= set(kept.tolist())           # window pinned
                # kept rows land in table[0..2] in original order
                tbl = lay.tables[r]
                for rank, t in enumerate(kept):
                    np.testing.assert_array_equal(
                        out.k_cache[l, tbl[rank // 4], rank % 4, h],
                        hw.k_cache[l, tbl[t // 4], t % 4, h])
        # reserved 4th block untouched
        np.testing.assert_array_equal(out.k_cache[:, lay.tables[r, 3]], hw.k_cache[:, lay.tables[r, 3]])
    # freed pushed on the stack
    assert out.fin.free_top == lay.free_top + 4
    assert list(out.fin.free_stack[lay.free_top:out.fin.free_top]) == list(out.fin.freed)


# ------------------------------------------------------------------ logits / softmax closed forms
def _rand_case(rng, G, w, d, b, T, h_kv=1):
    geo = O.Geometry(L=1, h_kv=h_kv, h_q=G * h_kv, d=d, b=b, N_total=-(-T // b) + 3, M=1, w=w, dtype="fp32")
    N = -(-T // b)
    table = rng.permutation(geo.N_total)[:N]
    q = rng.standard_normal((w, geo.h_q, d))
    k = rng.standard_normal((geo.N_total, b, h_kv, d))
    return geo, q, k, table


def test_single_head_single_query_is_textbook_softmax():
    """G=1, w=1: s = softmax(q K^T / sqrt(d)) over all t <= T-1 (scipy.special.softmax)."""
    rng = np.random.default_rng(0)
    geo, q, k, table = _rand_case(rng, G=1, w=1, d=8, b=4, T=11)
    T = 11
    s = O.attention_scores(O.logits_blockwise(geo, q, k, table, T, 0), T)
    Kd = np.stack([k[table[t // 4], t % 4, 0] for t in range(T)])
    ref = sp_softmax(Kd @ q[0, 0] / math.sqrt(8))
    np.testing.assert_allclose(s, ref, rtol=1e-12)


def test_hand_worked_logits():
    """d=2, b=2, T=3, w=1, G=1 worked by hand: q=(1,2), keys (1,0),(0,1),(1,1):
    logits (1, 2, 3)/sqrt(2); s = e^{x_t}/sum e^{x}."""
    geo = O.Geometry(L=1, h_kv=1, h_q=1, d=2, b=2, N_total=3, M=1, w=1, dtype="fp32")
    q = np.array([[[1.0, 2.0]]])
    k = np.zeros((3, 2, 1, 2))
    table = [2, 0]                       # logical block 0 -> physical 2, block 1 -> physical 0
    k[2, 0, 0] = [1, 0]; k[2, 1, 0] = [0, 1]; k[0, 0, 0] = [1, 1]
    s = O.attention_scores(O.logits_blockwise(geo, q, k, table, 3, 0), 3)
    x = [1 / math.sqrt(2), 2 / math.sqrt(2), 3 / math.sqrt(2)]
    e = [math.exp(v) for v in x]
    np.testing.assert_allclose(s, [v / sum(e) for v in e], rtol=1e-14)


@pytest.mark.parametrize("G,w,b,T", [(1, 3, 4, 10), (2, 4, 4, 13), (3, 2, 8, 17)])
def test_constant_keys_closed_form(G, w, b, T):
    """All K rows equal: P[g,u,t] = 1/(T-w+u+1) for t <= T-w+u, so
    s[t] = (1/w) * sum_{u: t <= T-w+u} 1/(T-w+u+1)."""
    rng = np.random.default_rng(1)
    geo, q, k, table = _rand_case(rng, G, w, 16, b, T)
    k[:] = rng.standard_normal(16)
    s = O.attention_scores(O.logits_dense(geo, q, k, table, T, 0), T)
    ref = np.array([sum(1.0 / (T - w + u + 1) for u in range(w) if t <= T - w + u) / w for t in range(T)])
    np.testing.assert_allclose(s, ref, rtol=1e-12)


def test_sum_rules_and_gqa_dominance():
    """G=1 => sum_t s = 1; G>1 => 1 <= sum s <= G; s >= each head's mean softmax."""
    rng = np.random.default_rng(2)
    geo, q, k, table = _rand_case(rng, 1, 4, 8, 4, 14)
    s = O.attention_scores(O.logits_dense(geo, q, k, table, 14, 0), 14)
    assert abs(s.sum() - 1) < 1e-12
    geo, q, k, table = _rand_case(rng, 3, 4, 8, 4, 14)
    A = O.logits_dense(geo, q, k, table, 14, 0)
    s = O.attention_scores(A, 14)
    assert 1 - 1e-12 <= s.sum() <= 3 + 1e-12
    for g in range(3):
        sg = O.attention_scores(A[g:g + 1], 14)
        assert np.all(s >= sg - 1e-15)


def test_identical_heads_equal_single_head():
    rng = np.random.default_rng(3)
    geo, q, k, table = _rand_case(rng, 3, 2, 8, 4, 9)
    q[:, 1] = q[:, 0]; q[:, 2] = q[:, 0]
    s3 = O.attention_scores(O.logits_dense(geo, q, k, table, 9, 0), 9)
    s1 = O.attention_scores(O.logits_dense(geo, q, k, table, 9, 0)[:1], 9)
    np.testing.assert_allclose(s3, s1, rtol=0, atol=0)


def test_max_over_heads_before_mean_over_window():
    """PAPER.md:409-411 order: softmax -> max over the GQA group -> mean over w.
    Two heads that attend one-hot to opposite tokens in each window row give s = [1, 1, 0, 0]
    (mean-then-max would give [0.5, 0.5, 0, 0])."""
    geo = O.Geometry(L=1, h_kv=1, h_q=2, d=2, b=4, N_total=1, M=1, w=2, dtype="fp32")
    k = np.zeros((1, 4, 1, 2))
    k[0, 0, 0] = [1000, 0]; k[0, 1, 0] = [0, 1000]
    c = math.sqrt(2)
    q = np.zeros((2, 2, 2))
    q[0, 0] = [c, -c]; q[0, 1] = [-c, c]        # row u=0: head0 -> t0, head1 -> t1
    q[1, 0] = [-c, c]; q[1, 1] = [c, -c]        # row u=1: head0 -> t1, head1 -> t0
    s = O.attention_scores(O.logits_blockwise(geo, q, k, [0], 4, 0), 4)
    np.testing.assert_array_equal(s, [1.0, 1.0, 0.0, 0.0])


def test_spec_mask_example():
    """SPEC.md:229 restated: w=2, b=4, last block: row 0 masks {3}, row 1 none (R1)."""
    geo = O.Geometry(L=1, h_kv=1, h_q=1, d=4, b=4, N_total=1, M=1, w=2, dtype="fp32")
    q = np.ones((2, 1, 4)); k = np.ones((1, 4, 1, 4))
    A = O.logits_blockwise(geo, q, k, [0], 4, 0)
    assert list(np.where(np.isinf(A[0, 0]))[0]) == [3]
    assert not np.isinf(A[0, 1]).any()


def test_blockwise_equals_dense():
    rng = np.random.default_rng(4)
    for G, w, b, T in [(2, 3, 4, 13), (1, 5, 2, 9), (4, 2, 8, 31)]:
        geo, q, k, table = _rand_case(rng, G, w, 8, b, T, h_kv=2)
        for h in range(2):
            A1 = O.logits_blockwise(geo, q, k, table, T, h)[:, :, :T]
            A2 = O.logits_dense(geo, q, k, table, T, h)
            np.testing.assert_allclose(A1, A2, rtol=1e-13, atol=1e-13)


# ------------------------------------------------------------------ pool / pin / select
def test_maxpool_spec_examples():
    np.testing.assert_array_equal(O.max_pool(np.array([1., 5., 2.]), 3), [5, 5, 5])
    np.testing.assert_array_equal(O.max_pool(np.array([0., 0., 9., 0., 0.]), 3), [0, 9, 9, 9, 0])
    x = np.random.default_rng(5).random(20)
    np.testing.assert_array_equal(O.max_pool(x, 1), x)
    assert np.all(O.max_pool(x, 7) >= x)
    # k=5 neighbourhood by hand at the edges: [a0..a2] and [a17..a19]
    assert O.max_pool(x, 5)[0] == x[:3].max() and O.max_pool(x, 5)[19] == x[17:].max()


def test_select_spec_examples():
    assert O.select(np.array([0.1, 0.9, 0.2, np.inf]), 2).tolist() == [1, 3]
    assert O.select(np.full(6, 0.5), 2).tolist() == [4, 5]      # ties -> newer wins (R7)
    assert O.select(np.arange(5.0), 5).tolist() == [0, 1, 2, 3, 4]


def test_select_brute_force():
    """Exhaustive enumeration of ell-subsets for T <= 10: the kept set is the subset whose
    descending (score, position) key list is lexicographically largest."""
    rng = np.random.default_rng(6)
    for trial in range(40):
        T = int(rng.integers(3, 11))
        ell = int(rng.integers(1, T + 1))
        s = rng.integers(0, 4, T).astype(float)        # many exact ties
        best = max(itertools.combinations(range(T), ell),
                   key=lambda sub: sorted(((s[t], t) for t in sub), reverse=True))
        assert O.select(s, ell).tolist() == sorted(best)


def test_window_always_kept():
    rng = np.random.default_rng(7)
    for _ in range(20):
        T, w = 30, 5
        s = O.pin_window(rng.random(T) * 1e30, T, w)
        assert set(range(T - w, T)) <= set(O.select(s, w).tolist())


# ------------------------------------------------------------------ compaction
def test_alg4_hand_trace():
    """SPEC.md:389 restated: b=2, kept {1,3} -> target slot 0 = old 1, slot 1 = old 3."""
    K = np.arange(4 * 2 * 1 * 1, dtype=np.float32).reshape(4, 2, 1, 1)
    V = -K.copy()
    table = [2, 0]
    tag = O.kept_to_tag(np.array([1, 3]), 2, 2)
    K0 = K.copy()
    O.compact_alg4(K, V, table, [2], tag, 0, 2)
    assert K[2, 0, 0, 0] == K0[2, 1, 0, 0] and K[2, 1, 0, 0] == K0[0, 1, 0, 0]
    assert V[2, 0, 0, 0] == -K0[2, 1, 0, 0]


def test_alg4_identity_and_equals_gather():
    rng = np.random.default_rng(8)
    for _ in range(30):
        b = int(rng.integers(1, 6)); N = int(rng.integers(3, 8)); nmax = int(rng.integers(2, N + 1))
        NT = N + 5
        K = rng.standard_normal((NT, b, 2, 3)).astype(np.float32); V = rng.standard_normal(K.shape).astype(np.float32)
        table = rng.permutation(NT)[:N]
        T = N * b - int(rng.integers(0, b))
        ell = int(rng.integers(1, min(T, (nmax - 1) * b) + 1))
        kept = np.sort(rng.choice(T, ell, replace=False))
        n_fresh = int(rng.integers(0, nmax))
        fresh = [x for x in range(NT) if x not in table][:n_fresh]
        targets = list(fresh) + list(table[len(fresh):nmax - 1])
        K1, V1, K2, V2 = K.copy(), V.copy(), K.copy(), V.copy()
        O.compact_alg4(K1, V1, table, targets, O.kept_to_tag(kept, N, b), 1, b)
        O.compact_gather(K2, V2, table, targets, kept, 1, b)
        np.testing.assert_array_equal(K1, K2); np.testing.assert_array_equal(V1, V2)
        # only head 1 rows of targets changed, and only ranks < ell
        changed = np.argwhere(np.any(K1 != K, axis=-1))
        for blk, slot, h in changed:
            assert h == 1 and blk in targets
            assert targets.index(blk) * b + slot < ell
    # identity: kept = {0..ell-1} with own targets => bytes unchanged
    K = rng.standard_normal((6, 4, 1, 2)); V = K.copy(); K0 = K.copy()
    O.compact_alg4(K, V, [0, 1, 2, 3], [0, 1, 2], O.kept_to_tag(np.arange(10), 4, 4), 0, 4)
    np.testing.assert_array_equal(K, K0)


# ------------------------------------------------------------------ planning / bookkeeping
def _plan_case(n_prefix, N=8, nmax=4, b=4):
    geo = O.Geometry(L=1, h_kv=1, h_q=1, d=2, b=b, N_total=40, M=1, w=2, dtype="fp32")
    prm = O.Params(n_max=nmax, flags=O.F_PREFIX)
    tables = np.arange(10, 10 + N, dtype=np.int32)[None, :]
    refs = np.zeros(40, np.int32); refs[tables[0]] = 1; refs[tables[0, :n_prefix]] = 3
    stack = np.zeros(40, np.int32); stack[:10] = np.arange(30, 40)
    return geo, prm, tables, refs, stack


@pytest.mark.parametrize("n_prefix,fresh,reused", [(0, 0, 3), (5, 3, 0), (2, 2, 1)])
def test_plan_targets_spec_cases(n_prefix, fresh, reused):
    """SPEC.md:397-399 restated (N_max=4): N_prefix=0 -> in place; 5 -> 3 fresh; 2 -> 2 fresh + 1 own."""
    geo, prm, tables, refs, stack = _plan_case(n_prefix)
    pl = O.plan(geo, prm, np.array([32]), tables, np.full((1, 1, 1), 8), refs, stack, 10)
    assert pl.status == O.OK
    t = pl.targets[0].tolist()
    assert t[:fresh] == [39, 38, 37][:fresh]                 # popped from the top
    assert t[fresh:] == tables[0, fresh:3].tolist()          # own blocks at the same index
    assert pl.reserved[0] == tables[0, max(n_prefix, 3)]
    fin = O.finalize(geo, prm, pl, tables, refs, stack, 10)
    assert fin.tables[0, :4].tolist() == t + [pl.reserved[0]]
    assert fin.ref_counts[tables[0, :n_prefix]].tolist() == [2] * n_prefix


def test_plan_errors():
    geo, prm, tables, refs, stack = _plan_case(0)
    bud = np.full((1, 1, 1), 8)
    assert O.plan(geo, prm, np.array([12]), tables, bud, refs, stack, 10).status == O.ERR_NOT_TRIGGERED
    assert O.plan(geo, prm, np.array([32]), tables, np.full((1, 1, 1), 1), refs, stack, 10).status == O.ERR_BAD_BUDGET
    assert O.plan(geo, prm, np.array([32]), tables, np.full((1, 1, 1), 13), refs, stack, 10).status == O.ERR_BAD_BUDGET
    geo, prm, tables, refs, stack = _plan_case(5)
    assert O.plan(geo, prm, np.array([32]), tables, bud, refs, stack, 2).status == O.ERR_NO_FREE_BLOCKS
    refs[tables[0, 6]] = 2   # shared block after a private one
    assert O.plan(geo, prm, np.array([32]), tables, bud, refs, stack, 10).status == O.ERR_BAD_TABLE
    t2 = tables.copy(); t2[0, 3] = 99
    assert O.plan(geo, O.Params(n_max=4), np.array([32]), t2, bud, None, stack, 10).status == O.ERR_BAD_TABLE


def test_plan_capacity_by_hand():
    """R18 on the Fig. 1 structure: A has N = 5, B has N = 7 blocks, b = 4,
    N_max = 4, no sharing -> the call frees 1 + 3 = 4 private blocks and pops none. The freed list needs
    4 entries; the free stack, with top = 4, grows to 4 + 4 = 8. One entry less in either buffer is
    ZPC_ERR_CAPACITY, checked before anything else is planned."""
    geo = O.Geometry(L=1, h_kv=1, h_q=1, d=2, b=4, N_total=16, M=2, w=2, dtype="fp32")
    prm = O.Params(n_max=4)
    tables = np.array([[0, 1, 2, 3, 4, -1, -1], [5, 6, 7, 8, 9, 10, 11]], np.int32)
    stack = np.zeros(16, np.int32)
    stack[:4] = [12, 13, 14, 15]
    seq, bud = np.array([20, 25]), np.full((2, 1, 1), 12)
    run = lambda fc, dc: O.plan(geo, prm, seq, tables, bud, None, stack, 4, None, fc, dc).status  # noqa: E731
    assert run(8, 4) == O.OK
    assert run(8, 3) == O.ERR_CAPACITY          # freed list one short
    assert run(7, 4) == O.ERR_CAPACITY          # free stack one short
    assert run(None, None) == O.OK              # unchecked when the caller gives no capacities
    # with a prefix: 2 shared blocks held only by this batch (ref = 2 = their occurrences) are driven to 0
    # and freed too, so both buffers need 2 more entries; a third external reference keeps them alive
    t2 = np.array([[0, 1, 2, 3, 4, -1, -1], [0, 1, 7, 8, 9, 10, 11]], np.int32)
    refs = np.zeros(16, np.int32)
    refs[t2[t2 >= 0]] = 1
    refs[[0, 1]] = 2
    p2 = O.Params(n_max=4, flags=O.F_PREFIX)
    st2 = np.zeros(16, np.int32)
    st2[:6] = [5, 6, 12, 13, 14, 15]
    pl = O.plan(geo, p2, seq, t2, bud, refs, st2, 6, None, 100, 100)
    assert pl.status == O.OK
    n_fresh = sum(min(int(pl.n_prefix[r]), 3) for r in range(2)) + sum(
        1 for r in range(2) if max(int(pl.n_prefix[r]), 3) >= [5, 7][r])
    freed = (5 - 1 - 3) + (7 - 1 - 3) + 2      # private non-targets + the two zeroed shared blocks
    need_stack = 6 - n_fresh + freed
    run2 = lambda fc, dc, rf: O.plan(geo, p2, seq, t2, bud, rf, st2, 6, None, fc, dc).status  # noqa: E731
    assert run2(need_stack, freed, refs) == O.OK
    assert run2(need_stack, freed - 1, refs) == O.ERR_CAPACITY
    assert run2(need_stack - 1, freed, refs) == O.ERR_CAPACITY
    refs3 = refs.copy()
    refs3[[0, 1]] = 3                           # held outside the batch: not freed
    assert run2(need_stack - 2, freed - 2, refs3) == O.OK
    assert run2(need_stack - 2, freed - 3, refs3) == O.ERR_CAPACITY


def test_block_conservation_random():
    """No leak, no double free: new tables + freed + still-held shared +
    free stack after == old tables + free stack before, as multisets with no duplicates."""
    rng = np.random.default_rng(9)
    for trial in range(25):
        b, nmax = 2, int(rng.integers(2, 5))
        R = int(rng.integers(1, 4))
        npref = int(rng.integers(0, 6))
        Ns = [int(rng.integers(max(nmax, npref), npref + 8)) for _ in range(R)]
        Ns = [max(n, nmax) for n in Ns]
        NT = sum(Ns) + 30
        perm = rng.permutation(NT).astype(np.int32)
        prefix = perm[:npref]; cur = npref
        stride = max(Ns)
        tables = np.full((R, stride), -1, np.int32)
        for r in range(R):
            tables[r, :npref] = prefix
            tables[r, npref:Ns[r]] = perm[cur:cur + Ns[r] - npref]; cur += Ns[r] - npref
        free = perm[cur:]
        stack = np.zeros(NT, np.int32); stack[:len(free)] = free
        hold = int(rng.integers(0, 2))
        refs = np.zeros(NT, np.int32); refs[tables[tables >= 0]] = 1
        refs[prefix] = R + hold
        flags = O.F_PREFIX if R + hold > 1 else 0
        geo = O.Geometry(L=1, h_kv=1, h_q=1, d=2, b=b, N_total=NT, M=R, w=1, dtype="fp32")
        prm = O.Params(n_max=nmax, flags=flags)
        seq = np.array([n * b - int(rng.integers(0, b)) for n in Ns], np.int32)
        bud = np.full((R, 1, 1), (nmax - 1) * b, np.int32)
        pl = O.plan(geo, prm, seq, tables, bud, refs if flags else None, stack, len(free))
        assert pl.status == O.OK
        fin = O.finalize(geo, prm, pl, tables, refs if flags else None, stack, len(free))
        before = [x for r in range(R) for x in tables[r, :Ns[r]]]
        before = set(before) | set(free.tolist())
        after_tables = [x for r in range(R) for x in fin.tables[r, :nmax]]
        still_shared = set(prefix.tolist()) - set(fin.freed.tolist()) if (hold and npref) else set()
        after = after_tables + fin.freed.tolist()  # freed are now on the stack
        stack_after = fin.free_stack[:fin.free_top].tolist()
        # the stack holds exactly the untouched free blocks + the freed ones
        assert len(stack_after) == len(set(stack_after))
        assert set(stack_after) >= set(fin.freed.tolist())
        held = set(after_tables) | still_shared | set(stack_after)
        assert held == before
        # no block both in a new table and on the stack
        assert not (set(after_tables) & set(stack_after))
        if flags:
            for blk in range(NT):
                members = sum(blk in fin.tables[r, :nmax] for r in range(R))
                expect = members + (hold if blk in prefix and blk not in fin.freed else 0)
                if blk in prefix and blk not in after_tables:
                    expect = hold if blk not in fin.freed else 0
                assert fin.ref_counts[blk] == expect, (blk, members)


@pytest.mark.parametrize("prefix_tokens,seq", [(8, 24), (16, 28), (24, 24)])
def test_prefix_compress_structure(prefix_tokens, seq):
    """§4.5: shared prefix blocks are never written; kept rows land in
    the target sequence (fresh blocks first, then own blocks); shared refs drop by one."""
    cfg = scaled(CONFIGS["prefix"], L=2, h_kv=2, h_q=4, d=16, b=4, w=2, n_max=4, pool_kernel=3,
                 seq_lens=[seq] * 3, budget=(2, 12), prefix_tokens=prefix_tokens, free_slack=3)
    hw = make_host_workload(cfg, seed=5)
    lay = hw.layout
    geo = geo_of(cfg, lay)
    prm = O.Params(n_max=4, pool_kernel=3, flags=O.F_PREFIX | O.F_VALIDATE)
    out = O.compress(geo, prm, hw.k_cache, hw.v_cache, hw.q_cache, lay.q_slots, lay.seq_lens,
                     lay.tables, hw.budgets, lay.ref_counts, lay.free_stack, lay.free_top)
    assert out.status == O.OK
    npref = prefix_tokens // 4
    for blk in lay.prefix_blocks:
        np.testing.assert_array_equal(out.k_cache[:, blk], hw.k_cache[:, blk])
        assert out.fin.ref_counts[blk] == 3 + 1 - 3
    for r in range(3):
        tg = out.plan.targets[r]
        assert all(t not in lay.tables[r, :npref] for t in tg)
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                kept = out.kept[(r, l, h)]
                assert len(kept) == min(seq, hw.budgets[r, l, h]) == out.new_lens[r, l, h]
                for rank, t in enumerate(kept):
                    np.testing.assert_array_equal(out.v_cache[l, tg[rank // 4], rank % 4, h],
                                                  hw.v_cache[l, lay.tables[r, t // 4], t % 4, h])


def test_widen_known_answers():
    """bf16 widening by bit placement (the stored 16 bits are the top half of an fp32): known values,
    including the smallest subnormal 2^-133, signed zero, infinities and NaN; fp32 passes through."""
    bits = np.array([0x3F80, 0xC000, 0x0001, 0x3FC0, 0x8000, 0x7F80, 0xFF80, 0x7FC0, 0x4049, 0x0080], np.uint16)
    out = O.widen(bits, "bf16")
    np.testing.assert_array_equal(out[:5], [1.0, -2.0, 2.0 ** -133, 1.5, 0.0])
    assert np.signbit(out[4])
    assert out[5] == np.inf and out[6] == -np.inf and np.isnan(out[7])
    assert out[8] == 3.140625                          # 0x4049: 1.5703125 * 2
    assert out[9] == 2.0 ** -126                       # smallest normal
    f = np.array([1.5, -0.1, 3e-40], np.float32)
    np.testing.assert_array_equal(O.widen(f, "fp32"), f.astype(np.float64))


def test_unit_keys_gather_by_construction():
    """unit_keys returns row t = K[l, table[t // b], t % b, h]: a pool whose element 0 encodes
    (layer, block, slot, head) is read back through a scrambled table, and the same rows come out of
    logits_dense (G = 1, w = 1, q = e_0 * sqrt(d)) -- the two gathers agree."""
    L, NT, b, hk, d = 2, 9, 4, 3, 4
    k = np.zeros((L, NT, b, hk, d))
    for l in range(L):
        for blk in range(NT):
            for s in range(b):
                for h in range(hk):
                    k[l, blk, s, h, 0] = 10000 * l + 100 * blk + 10 * s + h
    table = [7, 2, 5, 0]
    T = 14
    geo = O.Geometry(L=L, h_kv=hk, h_q=hk, d=d, b=b, N_total=NT, M=1, w=1, dtype="fp32")
    for l in range(L):
        for h in range(hk):
            rows = O.unit_keys(geo, k, table, T, l, h)
            expect = [10000 * l + 100 * table[t // b] + 10 * (t % b) + h for t in range(T)]
            np.testing.assert_array_equal(rows[:, 0], expect)
            q = np.zeros((1, hk, d))
            q[0, h, 0] = np.sqrt(d)
            lg = O.logits_dense(geo, q, k[l], table, T, h)
            np.testing.assert_allclose(lg[0, 0], expect)
