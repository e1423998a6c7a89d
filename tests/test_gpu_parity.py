"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle on the same seeded inputs.

Rules: scores within 1e-3 relative; kept sets exact outside
the 1e-3 band around the oracle's ell-th score; GPU S through the oracle's select reproduces
the GPU kept list bit for bit; whole K/V pools, tables, freed list, free stack and ref counts
bit-exact against oracle compaction driven by the GPU's kept lists.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params
from zpc_inputs import CONFIGS, make_host_workload, scaled
from zpc_inputs.device import from_host, generate, to_host

from helpers import full_check, gpu_results, run_gpu, snapshot_inputs

pytestmark = pytest.mark.gpu


def _run(cfg, seed=0, flags=0, pool=None, stages=False, strict=True, max_seq_len=None):
    hw = make_host_workload(cfg, seed)
    w = from_host(hw, max_seq_len=max_seq_len)
    inp = snapshot_inputs(w)
    desc, params = run_gpu(w, flags=flags, pool=pool, stages=stages)
    res = gpu_results(w, desc, params)
    full_check(w, inp, res, pool=pool, strict_select=strict)
    return w, res


@pytest.mark.parametrize("pool", [1, 3])
def test_fig1_toy(cuda_ok, pool):
    """BASELINE configs[0]: the Fig. 1 toy (fp32, CUDA-core scoring)."""
    cfg = scaled(CONFIGS["toy"], pool_kernel=pool)
    w, res = _run(cfg, seed=1, pool=pool)
    lay = w.layout
    A, B = lay.tables[0], lay.tables[1]
    assert res["freed"].tolist() == [A[4], B[4], B[5], B[6]]


def test_toy_stagewise_equals_fused(cuda_ok):
    cfg = CONFIGS["toy"]
    _run(cfg, seed=2, stages=True)


SMALL7B = scaled(CONFIGS["qwen7b"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 257, 416, 129 + 128],
                 budget=128, free_slack=5)


@pytest.mark.parametrize("flags", [0, zipc.ZPC_F_SCORE_CUDACORE])
def test_qwen7b_shape_small(cuda_ok, flags):
    """7B head shape (G=7, w=32, d=128, b=16, bf16), ragged T spanning several 128-token tiles."""
    _run(SMALL7B, seed=3, flags=flags)


def test_llama8b_shape_mixed_budgets(cuda_ok):
    cfg = scaled(CONFIGS["llama8b"], L=2, h_kv=2, h_q=8, n_max=9, seq_lens=[513, 700, 1030], budget=(32, 128),
                 wave=0)
    _run(cfg, seed=4)


def test_qwen32b_shape_d64_variant(cuda_ok):
    cfg = scaled(CONFIGS["qwen32b"], L=2, h_kv=2, h_q=10, d=64, n_max=6, seq_lens=[200, 333], budget=80, wave=0)
    _run(cfg, seed=5)


def test_prefix_small(cuda_ok):
    """§4.5 shared prefix with the harness holding a reference: fresh targets + own reuse."""
    for npref_tok, seq in [(64, 300), (160, 400), (256, 300)]:
        cfg = scaled(CONFIGS["prefix"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[seq] * 3, prefix_tokens=npref_tok,
                     budget=128, wave=0, free_slack=4)
        _run(cfg, seed=6)


@pytest.mark.parametrize("kind", ["plain", "prefix"])
def test_single_request(cuda_ok, kind):
    """R = 1 takes the single-CTA plan / finalize kernels (k_plan_small, k_finalize_small)."""
    if kind == "plain":
        cfg = scaled(CONFIGS["qwen32b"], L=2, h_kv=2, h_q=10, d=64, n_max=6, seq_lens=[333], budget=80, wave=0)
    else:
        cfg = scaled(CONFIGS["prefix"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[400], prefix_tokens=160,
                     budget=128, wave=0, free_slack=4)
    _run(cfg, seed=13)


@pytest.mark.parametrize("flags", [0, zipc.ZPC_F_SCORE_CUDACORE])
def test_paper_operating_point_shape(cuda_ok, flags):
    """NEXT-3: b = 256, w = 16, N_max = 9 with the Qwen3-8B head shape (G = 4), ragged T
    around the steady state N_max * b (one partial block, one freed block)."""
    cfg = scaled(CONFIGS["paper_op"], L=2, h_kv=2, h_q=8, seq_lens=[2304, 2100, 2500], wave=0, free_slack=3)
    _run(cfg, seed=8, flags=flags)


def test_paper_op_short_units_empty_ranks(cuda_ok):
    """k_score_res sizes its cluster by the longest unit (T = 2500 -> 6 ranks); a short unit in the same call
    (T = 300: 3 tiles) leaves ranks without tiles, which must publish an empty (max, sum) and score nothing."""
    cfg = scaled(CONFIGS["paper_op"], L=2, h_kv=2, h_q=8, b=128, n_max=3, seq_lens=[300, 2500, 1000], budget=(16, 256),
                 wave=0, free_slack=4)
    w = from_host(make_host_workload(cfg, 9))
    desc, params = desc_params(w)
    assert zipc.zpc_score_path(desc, params) == zipc.ZPC_PATH_RESIDENT
    inp = snapshot_inputs(w)
    desc, params = run_gpu(w)
    full_check(w, inp, gpu_results(w, desc, params))


def test_paper_op_normaliser_overflow_path(cuda_ok):
    """k_score_res's one-sweep normaliser uses the logit of each warp's first token as the exp2 reference; a
    logit ~100 log2 units above it must send the unit to the exact max-then-sum path. Key rows scaled by 2^6
    (exact in bf16) make such logits; the oracle (fp64, max-subtracted softmax) must still be matched."""
    cfg = scaled(CONFIGS["paper_op"], L=1, h_kv=2, h_q=8, seq_lens=[2304, 2100], wave=0, free_slack=3)
    hw = make_host_workload(cfg, 5)
    lay = hw.layout
    for t in (700, 1500):                                  # inside slices, never a warp's first token
        blk, slot = lay.tables[0, t // cfg.b], t % cfg.b
        row = hw.k_cache[0, blk, slot, 0].astype(np.uint32) << 16
        f = (row.view(np.float32) * 64.0).astype(np.float32)
        hw.k_cache[0, blk, slot, 0] = (f.view(np.uint32) >> 16).astype(np.uint16)
    w = from_host(hw)
    inp = snapshot_inputs(w)
    desc, params = run_gpu(w)
    assert zipc.zpc_score_path(desc, params) == zipc.ZPC_PATH_RESIDENT
    full_check(w, inp, gpu_results(w, desc, params))


def test_paper_operating_point_g8(cuda_ok):
    """w = 16 with G = 8 (Qwen3-32B-like head ratio), tcgen05 path."""
    cfg = scaled(CONFIGS["paper_op"], L=1, h_kv=2, h_q=16, seq_lens=[2304, 2049], wave=0, free_slack=3)
    _run(cfg, seed=9)


def test_edge_min_trigger_and_w_gt_b(cuda_ok):
    """N == N_max exactly, partial last block, w > b, budget == w."""
    cfg = scaled(CONFIGS["qwen7b"], L=1, h_kv=1, h_q=7, n_max=3, seq_lens=[33, 48, 40], budget=32, free_slack=2)
    _run(cfg, seed=7)


def test_generator_device_equals_host(cuda_ok):
    cfg = scaled(CONFIGS["prefix"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[300] * 2, prefix_tokens=64, wave=0)
    hw = make_host_workload(cfg, 11)
    dw = generate(cfg, 11, np.arange(2))
    np.testing.assert_array_equal(to_host(dw.k, True), hw.k_cache)
    np.testing.assert_array_equal(to_host(dw.v, True), hw.v_cache)
    np.testing.assert_array_equal(to_host(dw.q, True), hw.q_cache)


@pytest.mark.parametrize("case", ["not_triggered", "bad_budget", "no_free", "bad_slot", "bad_table", "capacity",
                                  "nonfinite_k", "nonfinite_q"])
def test_device_errors_mutate_nothing(cuda_ok, case):
    cfg = scaled(CONFIGS["prefix"], L=1, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 300], prefix_tokens=64,
                 budget=128, wave=0, free_slack=4)
    hw = make_host_workload(cfg, 8)
    expect = {"not_triggered": zipc.ZPC_ERR_NOT_TRIGGERED, "bad_budget": zipc.ZPC_ERR_BAD_BUDGET,
              "no_free": zipc.ZPC_ERR_NO_FREE_BLOCKS, "bad_slot": zipc.ZPC_ERR_BAD_SLOT,
              "bad_table": zipc.ZPC_ERR_BAD_TABLE, "capacity": zipc.ZPC_ERR_CAPACITY,
              "nonfinite_k": zipc.ZPC_ERR_NONFINITE, "nonfinite_q": zipc.ZPC_ERR_NONFINITE}[case]
    lay = hw.layout
    flags = zipc.ZPC_F_VALIDATE if case.startswith("nonfinite") else 0
    if case == "nonfinite_k":   # one key element of request 1, layer 0, head 1, token 137 -> bf16 NaN
        t = 137
        hw.k_cache[0, lay.tables[1, t // cfg.b], t % cfg.b, 1, 5] = 0x7FC0
    elif case == "nonfinite_q":   # a window query element of request 0 (head group of KV head 0) -> +inf
        hw.q_cache[0, lay.q_slots[0], 3, 2, 7] = 0x7F80
    if case == "not_triggered":
        lay.seq_lens[1] = 16 * 8
    elif case == "bad_budget":
        hw.budgets[1, 0, 1] = 8 * 16 + 1
    elif case == "no_free":
        lay.free_top = 3
    elif case == "bad_slot":
        lay.q_slots[0] = lay.M
    elif case == "bad_table":
        lay.tables[1, 10] = lay.N_total
    w = from_host(hw)
    if case == "capacity":   # a freed-list buffer one entry shorter than the blocks the call frees
        need = sum(int(np.ceil(T / cfg.b)) - 1 - (cfg.n_max - 1) for T in lay.seq_lens) + 0
        w.freed = w.freed[:need - 1].clone()
    before = snapshot_inputs(w)
    desc, params = run_gpu(w, flags=flags)
    assert int(w.status.item()) == expect
    np.testing.assert_array_equal(to_host(w.k, True), before["k"])
    np.testing.assert_array_equal(to_host(w.tables), before["tables"])
    np.testing.assert_array_equal(to_host(w.free_stack), before["stack"])
    assert int(w.free_top.item()) == before["top"]
    np.testing.assert_array_equal(to_host(w.ref_counts), before["refs"])
    # oracle agrees on the code
    geo = O.Geometry(cfg.L, cfg.h_kv, cfg.h_q, cfg.d, cfg.b, lay.N_total, lay.M, cfg.w, cfg.dtype)
    prm = O.Params(cfg.n_max, flags=O.F_PREFIX | (O.F_VALIDATE if flags else 0), max_seq_len=w.max_seq_len)
    ref = O.compress(geo, prm, before["k"], before["v"], before["q"], before["slots"], before["seq"],
                     before["tables"], before["budgets"], before["refs"], before["stack"], before["top"],
                     free_capacity=len(before["stack"]), freed_capacity=int(w.freed.numel()))
    assert ref.status == expect


@pytest.mark.parametrize("mapped", [False, True])
def test_host_variant_equals_device(cuda_ok, mapped):
    """zpc_compress_host (host bookkeeping, copies inside the call; with ZPC_F_HOST_MAPPED one gather and one
    scatter kernel on the pinned host arrays) == zpc_compress."""
    hw = make_host_workload(SMALL7B, 9)
    w1 = from_host(hw)
    run_gpu(w1)
    w2 = from_host(hw)
    desc, params = desc_params(w2)
    if mapped:
        params.flags |= zipc.ZPC_F_HOST_MAPPED
    R = int(w2.seq_lens.numel())
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    host = {k: pin(getattr(w2, k)) for k in ("q_slots", "seq_lens", "tables", "budgets", "new_lens",
                                            "new_num_blocks", "free_stack", "free_top", "freed", "num_freed",
                                            "status")}
    need = zipc.zpc_workspace_bytes_host(desc, params, R, host["tables"].shape[1], host["free_stack"].numel(),
                                         host["freed"].numel())
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    b = zipc.make_batch(k_cache=w2.k, v_cache=w2.v, q_cache=w2.q, q_slots=host["q_slots"],
                        seq_lens=host["seq_lens"], block_tables=host["tables"], budgets=host["budgets"],
                        new_lens=host["new_lens"], new_num_blocks=host["new_num_blocks"], ref_counts=None,
                        free_stack=host["free_stack"], free_top=host["free_top"], freed_blocks=host["freed"],
                        num_freed=host["num_freed"], workspace=ws, status=host["status"])
    zipc.zpc_compress_host(desc, params, b)
    torch.cuda.synchronize()
    assert int(host["status"][0]) == 0
    assert torch.equal(w1.k.cpu(), w2.k.cpu()) and torch.equal(w1.v.cpu(), w2.v.cpu())
    assert torch.equal(w1.tables.cpu(), host["tables"])
    n = int(host["num_freed"][0])
    assert n == int(w1.num_freed.item())
    assert torch.equal(w1.freed.cpu()[:n], host["freed"][:n])
    assert torch.equal(w1.new_lens.cpu(), host["new_lens"])


@pytest.mark.parametrize("mapped", [False, True])
def test_host_variant_prefix(cuda_ok, mapped):
    """zpc_compress_host with shared-prefix ref counts: fresh pops, freed shared blocks and the
    ref-count updates come back to the host arrays identical to the device-resident call, with per-array copies
    or with the ZPC_F_HOST_MAPPED gather / scatter kernels."""
    cfg = scaled(CONFIGS["prefix"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[400] * 3, prefix_tokens=160,
                 budget=128, wave=0, free_slack=4)
    hw = make_host_workload(cfg, 12)
    w1 = from_host(hw)
    run_gpu(w1)
    w2 = from_host(hw)
    desc, params = desc_params(w2)
    assert params.flags & zipc.ZPC_F_PREFIX
    if mapped:
        params.flags |= zipc.ZPC_F_HOST_MAPPED
    R = int(w2.seq_lens.numel())
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    host = {k: pin(getattr(w2, k)) for k in ("q_slots", "seq_lens", "tables", "budgets", "new_lens",
                                            "new_num_blocks", "ref_counts", "free_stack", "free_top", "freed",
                                            "num_freed", "status")}
    need = zipc.zpc_workspace_bytes_host(desc, params, R, host["tables"].shape[1], host["free_stack"].numel(),
                                         host["freed"].numel())
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    b = zipc.make_batch(k_cache=w2.k, v_cache=w2.v, q_cache=w2.q, q_slots=host["q_slots"],
                        seq_lens=host["seq_lens"], block_tables=host["tables"], budgets=host["budgets"],
                        new_lens=host["new_lens"], new_num_blocks=host["new_num_blocks"], ref_counts=host["ref_counts"],
                        free_stack=host["free_stack"], free_top=host["free_top"], freed_blocks=host["freed"],
                        num_freed=host["num_freed"], workspace=ws, status=host["status"])
    zipc.zpc_compress_host(desc, params, b)
    torch.cuda.synchronize()
    assert int(host["status"][0]) == 0
    assert torch.equal(w1.k.cpu(), w2.k.cpu()) and torch.equal(w1.v.cpu(), w2.v.cpu())
    assert torch.equal(w1.tables.cpu(), host["tables"])
    assert torch.equal(w1.ref_counts.cpu(), host["ref_counts"])
    assert torch.equal(w1.free_stack.cpu(), host["free_stack"]) and int(w1.free_top.item()) == int(host["free_top"][0])
    n = int(host["num_freed"][0])
    assert n == int(w1.num_freed.item())
    assert torch.equal(w1.freed.cpu()[:n], host["freed"][:n])
    assert torch.equal(w1.new_lens.cpu(), host["new_lens"])
    assert torch.equal(w1.new_num_blocks.cpu(), host["new_num_blocks"])


def test_deterministic(cuda_ok):
    hw = make_host_workload(SMALL7B, 10)
    outs = []
    for _ in range(2):
        w = from_host(hw)
        desc, params = run_gpu(w)
        outs.append(gpu_results(w, desc, params))
    T = hw.layout.seq_lens
    cfg = SMALL7B
    for o in outs:   # only defined entries: S[:T] and kept[:ell] per unit
        for u in range(o["S"].shape[0]):
            r = u // (cfg.L * cfg.h_kv)
            o["S"][u, T[r]:] = 0
            o["kept"][u, o["new_lens"].reshape(-1)[u]:] = 0
        o["stack"] = o["stack"][:o["top"]]
    for key in ("S", "kept", "k", "v", "tables", "freed", "stack", "new_lens"):
        np.testing.assert_array_equal(outs[0][key], outs[1][key])


# Several units per persistent CTA cluster (192 units > the 74 clusters of a B200), so the overlapped
# schedule interleaves pass 1 of one unit with pass 2 of the previous one on every cluster, with ragged
# lengths (partial last tiles, a unit whose 256-token pair tile is half empty). "default" is the cooperative
# pair kernel for G = 5, 7, 8 and the overlapped kernel for G = 4; "serial" forces k_score_tc
# (params.variant ZPC_V_SCORE_SERIAL).
@pytest.mark.parametrize("variant", ["default", "serial"])
@pytest.mark.parametrize("shape", [("qwen7b", 7), ("qwen32b", 5), ("llama8b", 4), ("llama8b", 8)])
def test_many_units_per_cluster(cuda_ok, monkeypatch, variant, shape):
    name, G = shape
    monkeypatch.setattr(zipc, "DEFAULT_VARIANT", zipc.variant(score_serial=variant == "serial"))
    cfg = scaled(CONFIGS[name], L=4, h_kv=8, h_q=8 * G, n_max=9,
                 seq_lens=[300, 1100, 144, 700, 385, 896], budget=(32, 128), wave=0, free_slack=6)
    _run(cfg, seed=11 + G)


# k_score_coop with K tiles by TMA (blocks of >= 128 slots): b = 128 and 256, ragged lengths
@pytest.mark.parametrize("b,n_max", [(128, 5), (256, 3)])
def test_coop_tma_blocks(cuda_ok, b, n_max):
    cfg = scaled(CONFIGS["qwen7b"], L=2, h_kv=2, h_q=14, b=b, n_max=n_max, seq_lens=[1100, 700, 1500], budget=(32, 256),
                 wave=0, free_slack=4)
    w = from_host(make_host_workload(cfg, 60 + b))
    desc, params = desc_params(w)
    assert zipc.zpc_score_path(desc, params) == zipc.ZPC_PATH_COOP
    inp = snapshot_inputs(w)
    desc, params = run_gpu(w)
    full_check(w, inp, gpu_results(w, desc, params))


# MHA (G = 1) and the GQA ratios without a config (G = 2, 3, 6) on the tensor-core path (k_score_tc), at
# d = 128 and d = 64; the library reports which scoring kernel family a call takes (zpc_score_path)
@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("G", [1, 2, 3, 6])
def test_generic_gqa_ratios(cuda_ok, G, d):
    cfg = scaled(CONFIGS["qwen7b"], L=2, h_kv=4, h_q=4 * G, d=d, n_max=9, seq_lens=[300, 1100, 144, 385],
                 budget=(32, 128), wave=0, free_slack=6)
    w = from_host(make_host_workload(cfg, 40 + G))
    desc, params = desc_params(w)
    assert zipc.zpc_score_path(desc, params) == zipc.ZPC_PATH_TC
    inp = snapshot_inputs(w)
    desc, params = run_gpu(w)
    full_check(w, inp, gpu_results(w, desc, params))


# Long units (the first compression after a long prefill sees T far above N_max * b): 64K and
# 128K tokens with ragged lengths, past the 48K shared-memory select (k_select keys in the workspace), through
# the cooperative scoring kernel and the per-unit one
@pytest.mark.parametrize("variant", ["default", "serial"])
@pytest.mark.parametrize("seqs", [[65536 + 77, 50001], [131072 - 5, 70001]])
def test_long_units(cuda_ok, monkeypatch, variant, seqs):
    monkeypatch.setattr(zipc, "DEFAULT_VARIANT", zipc.variant(score_serial=variant == "serial"))
    cfg = scaled(CONFIGS["qwen7b"], L=1, h_kv=1, h_q=7, n_max=9, seq_lens=seqs, budget=(32, 128), wave=0,
                 free_slack=4)
    w = from_host(make_host_workload(cfg, 77))
    assert w.max_seq_len > 49152
    inp = snapshot_inputs(w)
    desc, params = run_gpu(w)
    full_check(w, inp, gpu_results(w, desc, params))


# k_select_reg at every thread-count instance: the dispatch follows the host bound max_seq_len, so small
# ragged units run through the 256 x 32 / 512 x 32 / 1024 x 32 variants (and k_select for comparison)
@pytest.mark.parametrize("max_seq_len,mode", [(2048, "2"), (8192, "1"), (16384, "1"), (32768, "1"), (8192, "0")])
def test_select_kernels(cuda_ok, monkeypatch, max_seq_len, mode):
    monkeypatch.setattr(zipc, "DEFAULT_VARIANT", zipc.variant(select={"0": 1, "1": 0, "2": 2}[mode]))
    cfg = scaled(CONFIGS["qwen7b"], L=2, h_kv=4, h_q=28, n_max=9, seq_lens=[300, 1100, 144, 700, 385],
                 budget=(32, 128), wave=0, free_slack=6, pool_kernel=7)
    _run(cfg, seed=21, max_seq_len=max_seq_len)


# k_select_reg's pooling has a register doubling tree for k_p = 7 and the direct loop for every other
# k_p: the other widths through the register kernel too (strict selection pins the pooled keys)
@pytest.mark.parametrize("pool", [1, 3, 5, 9])
def test_select_reg_other_pools(cuda_ok, monkeypatch, pool):
    monkeypatch.setattr(zipc, "DEFAULT_VARIANT", zipc.variant(select=2))
    cfg = scaled(CONFIGS["qwen7b"], L=1, h_kv=4, h_q=28, n_max=9, seq_lens=[300, 1100, 144, 385],
                 budget=(32, 128), wave=0, free_slack=6, pool_kernel=pool)
    _run(cfg, seed=23, pool=pool, max_seq_len=2048)


@pytest.mark.parametrize("nt", [128, 256, 512, 1024])
def test_compact_every_cta_width(cuda_ok, monkeypatch, nt):
    """k_compact at each CTA width launch_compact can pick (params.variant overrides the per-call choice):
    chunk = NT/VPR ranks, so the hazard ordering (reads of a chunk before its writes, kept[i] >= i) is
    exercised at 8..128 ranks per chunk, for VPR = 16 (bf16 d = 128) and VPR = 8 (bf16 d = 64)."""
    monkeypatch.setattr(zipc, "DEFAULT_VARIANT", zipc.variant(compact_nt=nt))
    _run(SMALL7B, seed=40 + nt)
    cfg = scaled(CONFIGS["qwen32b"], L=2, h_kv=2, h_q=10, d=64, n_max=6, seq_lens=[200, 333], budget=80, wave=0)
    _run(cfg, seed=41 + nt)


def test_pool_first_only(cuda_ok):
    """ZPC_F_POOL_FIRST (R32): requests compressed before select on the unpooled score,
    first-time requests on the k_p = 7 pooled one; every parity rule with the oracle doing the same."""
    cfg = scaled(CONFIGS["qwen7b"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 257, 416, 257], budget=128,
                 free_slack=5, pool_kernel=7)
    hw = make_host_workload(cfg, 13)
    hw.is_compressed = np.array([1, 0, 1, 0], np.int32)
    w = from_host(hw)
    inp = snapshot_inputs(w)
    desc, params = desc_params(w, flags=zipc.ZPC_F_POOL_FIRST)
    zipc.zpc_compress(desc, params, batch_of(w, desc, params))
    torch.cuda.synchronize()
    full_check(w, inp, gpu_results(w, desc, params), pool_first_compressed=hw.is_compressed)
