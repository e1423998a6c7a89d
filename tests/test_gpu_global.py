"""GPU parity of NEXT-2 (ZPC_F_GLOBAL_SCORE): Alg. 2 global score inside the
selection and F relocation with the kept rows, through the C ABI vs the fp64 oracle.

Rules: the workspace S (overwritten with the global score for compressed requests, Alg. 2 line 11)
within 1e-3 relative of the oracle's global score; kept sets by the band rule on the oracle's pooled
+pinned global score and exactly equal to the oracle's selection on the GPU's own S; the F pool after
the step equals the oracle's (Alg. 2 update, then relocation driven by the GPU's kept lists) --
untouched entries bit-exact, updated ones within 1e-3 relative; K/V bytes bit-exact.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params
from zpc_inputs import CONFIGS, global_history, make_host_workload, scaled
from zpc_inputs.device import from_host, to_host

from helpers import check_band, check_scores, geometry, gpu_results, snapshot_inputs, unit_index

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["select_auto", "select_reg"])
def _select_path(request, monkeypatch):
    """Run every case through both selection kernels: k_select (what these small T get by default)
    and the register-resident k_select_reg (params.variant select = 2 forces it for T <= 32K)."""
    monkeypatch.setattr(zipc, "DEFAULT_VARIANT", zipc.variant(select=2 if request.param == "select_reg" else 0))

ALPHA = 0.8
CASES = {
    "bf16_7b": scaled(CONFIGS["qwen7b"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[300, 257, 416, 129 + 128],
                      budget=128, free_slack=5),
    "fp32_toy": scaled(CONFIGS["toy"], pool_kernel=3),
    "bf16_8b_mixed": scaled(CONFIGS["llama8b"], L=2, h_kv=2, h_q=8, n_max=9, seq_lens=[513, 700, 1030],
                            budget=(32, 128), wave=0),
    # three requests sharing a 160-token prefix (10 blocks): R31, the shared blocks' F is read, not stored
    "bf16_prefix_shared": scaled(CONFIGS["prefix"], L=2, h_kv=2, h_q=14, n_max=9, seq_lens=[400] * 3,
                                 prefix_tokens=160, budget=128, wave=0, free_slack=4),
}


def _workload(cfg, seed, comp=None, scale=None):
    hw = make_host_workload(cfg, seed)
    f, c = global_history(cfg, seed, hw.layout.N_total, hw.layout.rids, scale=scale)
    hw.f_cache, hw.is_compressed = f, (c if comp is None else np.asarray(comp, np.int32))
    return hw


@pytest.mark.parametrize("name", list(CASES))
def test_global_score_parity(cuda_ok, name):
    cfg = CASES[name]
    hw = _workload(cfg, 31)
    w = from_host(hw)
    inp = snapshot_inputs(w)
    f0 = hw.f_cache.copy()
    desc, params = desc_params(w, global_alpha=ALPHA)
    zipc.zpc_compress(desc, params, batch_of(w, desc, params))
    torch.cuda.synchronize()
    res = gpu_results(w, desc, params)
    geo = geometry(w)
    flags = O.F_GLOBAL_SCORE | (O.F_PREFIX if w.layout.ref_counts is not None else 0)
    prm = O.Params(n_max=cfg.n_max, pool_kernel=cfg.pool_kernel, max_seq_len=w.max_seq_len, flags=flags, alpha=ALPHA)
    kw = dict(free_capacity=len(inp["stack"]), freed_capacity=len(to_host(w.freed)), f_cache=f0,
              is_compressed=hw.is_compressed)
    ref = O.compress(geo, prm, inp["k"], inp["v"], inp["q"], inp["slots"], inp["seq"], inp["tables"], inp["budgets"],
                     inp["refs"], inp["stack"], inp["top"], **kw)
    assert res["status"] == ref.status == O.OK
    gpu_kept = {}
    for r in range(len(inp["seq"])):
        T = int(inp["seq"][r])
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                key, u = (r, l, h), unit_index(w, r, l, h)
                where = f"{name} r={r} l={l} h={h} compressed={hw.is_compressed[r]}"
                check_scores(res["S"][u, :T], ref.global_scores[key], where)
                ell = int(res["new_lens"][r, l, h])
                kg = res["kept"][u, :ell].copy()
                gpu_kept[key] = kg
                check_band(kg, O.pin_window(O.max_pool(ref.global_scores[key], cfg.pool_kernel), T, cfg.w), ell, where)
                sel = O.select(O.pin_window(O.max_pool(res["S"][u, :T].astype(np.float64), cfg.pool_kernel), T,
                                            cfg.w), ell)
                np.testing.assert_array_equal(sel, kg, err_msg=where)
    ref2 = O.compress(geo, prm, inp["k"], inp["v"], inp["q"], inp["slots"], inp["seq"], inp["tables"],
                      inp["budgets"], inp["refs"], inp["stack"], inp["top"], kept_override=gpu_kept, **kw)
    np.testing.assert_array_equal(res["k"], ref2.k_cache)
    np.testing.assert_array_equal(res["v"], ref2.v_cache)
    np.testing.assert_array_equal(res["tables"], ref2.fin.tables)
    f_gpu = to_host(w.f_cache)
    same = ref2.f_cache == f0
    changed = ~same | (f_gpu != f0)
    np.testing.assert_array_equal(f_gpu[~changed], f0[~changed])
    np.testing.assert_allclose(f_gpu[changed], ref2.f_cache[changed], rtol=1e-3, atol=1e-30)


def test_uncompressed_batch_selects_like_plain_method(cuda_ok):
    cfg = CASES["bf16_7b"]
    hw = _workload(cfg, 32, comp=np.zeros(len(cfg.seq_lens), np.int32))
    outs = []
    for ga in (None, ALPHA):
        w = from_host(hw)
        desc, params = desc_params(w, global_alpha=ga)
        zipc.zpc_compress(desc, params, batch_of(w, desc, params))
        torch.cuda.synchronize()
        outs.append((to_host(w.new_lens), to_host(w.k, True), to_host(w.tables), w))
    for a, b in zip(outs[0][:3], outs[1][:3]):
        np.testing.assert_array_equal(a, b)


def test_global_requires_pool_pointers(cuda_ok):
    cfg = CASES["bf16_7b"]
    w = from_host(make_host_workload(cfg, 33))      # no f_cache / is_compressed
    desc, params = desc_params(w, global_alpha=ALPHA)
    with pytest.raises(zipc.ZipcError):
        zipc.zpc_compress(desc, params, batch_of(w, desc, params))
