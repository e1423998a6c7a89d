"""Full-size parity for the other BASELINE configs, each in the launch configuration bench.py times
(`python bench.py --config NAME`: the config's per-GPU wave of global request ids 0..wave-1, seed 2603):

* llama8b  (configs[2]): 32 requests x 16384 tokens, G = 4, mixed per-head budgets U{32..2048};
* qwen32b  (configs[3]): 16 requests x 32768 tokens, G = 5 (~137 GB of K/V: one config alive at a time);
* prefix   (configs[4]): 128 requests x (4096 shared + 8192 private) tokens, fresh targets, ref counts.

Sampled units are checked against the oracle on host-regenerated inputs (never read back from the GPU
generator): scores within 1e-3, the band rule, the strict select of the GPU's own S, and the K/V bytes at
every kept rank in the request's NEW table (fresh targets included). Every unit's kept list is checked
for order, length and the pinned window; every request's table / freed-list structure for the
config's a0/a6 rules."""
import gc

import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_08743_b200 import zipc
from paper_2603_08743_b200.batch import batch_of, desc_params, workspace_view
from zpc_inputs import CONFIGS, k_rows, q_rows, v_rows
from zpc_inputs.device import generate

from helpers import check_band, check_scores

pytestmark = pytest.mark.gpu
SEED = 2603


@pytest.fixture(scope="module", params=["llama8b", "qwen32b", "prefix"])
def run_cfg(request):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CONFIGS[request.param]
    wave = cfg.wave or cfg.R
    w = generate(cfg, SEED, np.arange(wave))
    tables0 = w.layout.tables.copy()
    refs0 = None if w.layout.ref_counts is None else w.layout.ref_counts.copy()
    desc, params = desc_params(w, flags=zipc.ZPC_F_COUNT_MOVES)
    zipc.zpc_compress(desc, params, batch_of(w, desc, params))
    torch.cuda.synchronize()
    yield cfg, w, desc, params, tables0, refs0
    del w
    gc.collect()
    torch.cuda.empty_cache()


def _samples(cfg, R):
    return [(0, 0, 0), (R - 1, cfg.L - 1, cfg.h_kv - 1), (R // 2, cfg.L // 3, min(1, cfg.h_kv - 1))]


def test_structure(run_cfg):
    cfg, w, desc, params, tables0, refs0 = run_cfg
    assert int(w.status.item()) == 0
    R = len(w.layout.seq_lens)
    T = w.layout.seq_lens.astype(np.int64)
    nm = cfg.n_max
    np.testing.assert_array_equal(w.new_lens.cpu().numpy(), np.minimum(T[:, None, None], w.budgets_host))
    assert (w.new_num_blocks.cpu().numpy() == nm).all()
    tables = w.tables.cpu().numpy()
    npre = cfg.prefix_tokens // cfg.b
    if npre == 0:
        # in place: the first N_max entries stay the request's own first N_max blocks; the
        # rest are freed in ascending logical order, requests in input order
        np.testing.assert_array_equal(tables[:, :nm], tables0[:, :nm])
        N = -(-T // cfg.b)
        expect = np.concatenate([tables0[r, nm:N[r]] for r in range(R)])
        freed = w.freed.cpu().numpy()[:int(w.num_freed.item())]
        np.testing.assert_array_equal(freed, expect)
    else:
        # N_prefix >= N_max - 1: every target is a fresh block, none of them shared or own
        refs = w.ref_counts.cpu().numpy()
        fresh = tables[:, :nm - 1]
        assert len(np.unique(fresh)) == fresh.size, "a fresh target handed out twice"
        for r in range(R):
            assert not set(fresh[r].tolist()) & set(tables0[r, :-(-int(T[r]) // cfg.b)].tolist())
        # shared prefix blocks lost one reference per request
        pre = tables0[0, :npre]
        np.testing.assert_array_equal(refs[pre], refs0[pre] - R)


def test_kept_lists_all_units(run_cfg):
    cfg, w, desc, params, tables0, refs0 = run_cfg
    R = len(w.layout.seq_lens)
    lay = zipc.zpc_workspace_layout_get(desc, params, R)
    units = R * cfg.L * cfg.h_kv
    kept = workspace_view(w, desc, params, "kept", torch.int32, (units, lay.kept_stride))
    ell = w.new_lens.reshape(-1).long()
    T = torch.from_numpy(np.repeat(w.layout.seq_lens.astype(np.int64), cfg.L * cfg.h_kv)).to(kept.device)
    rng = torch.arange(lay.kept_stride, device=kept.device)
    valid = rng[None, :] < ell[:, None]
    k = torch.where(valid, kept.long(), T[:, None])
    assert bool(((k[:, 1:] > k[:, :-1]) | ~valid[:, 1:]).all())
    assert bool(((k >= 0) & (k <= T[:, None])).all())
    last = torch.gather(kept, 1, (ell[:, None] - cfg.w + torch.arange(cfg.w, device=kept.device)[None, :]))
    assert bool((last.long() == (T[:, None] - cfg.w + torch.arange(cfg.w, device=kept.device)[None, :])).all())


@pytest.mark.parametrize("k", range(3))
def test_sampled_units_vs_oracle(run_cfg, k):
    cfg, w, desc, params, tables0, refs0 = run_cfg
    R = len(w.layout.seq_lens)
    r, l, h = _samples(cfg, R)[k]
    T = int(w.layout.seq_lens[r])
    kt = k_rows(cfg, SEED, r, l, h, np.arange(T), T)                 # bf16 bits [T, d], logical order
    q = q_rows(cfg, SEED, r, l)
    N = -(-T // cfg.b)
    kpad = np.zeros((N * cfg.b, cfg.d), kt.dtype)
    kpad[:T] = kt
    geo = O.Geometry(L=1, h_kv=1, h_q=cfg.G, d=cfg.d, b=cfg.b, N_total=N, M=1, w=cfg.w, dtype="bf16")
    kf = O.widen(kpad, "bf16").reshape(N, cfg.b, 1, cfg.d)
    qf = O.widen(q[:, h * cfg.G:(h + 1) * cfg.G, :], "bf16")
    s_ref = O.attention_scores(O.logits_dense(geo, qf, kf, np.arange(N), T, 0), T)
    units = R * cfg.L * cfg.h_kv
    lay = zipc.zpc_workspace_layout_get(desc, params, R)
    u = (r * cfg.L + l) * cfg.h_kv + h
    where = f"{cfg.name} unit {r},{l},{h}"
    S = workspace_view(w, desc, params, "scores", torch.float32, (units, w.max_seq_len))[u, :T].cpu().numpy()
    check_scores(S, s_ref, where)
    ell = int(w.new_lens[r, l, h].item())
    assert ell == min(T, int(w.budgets_host[r, l, h]))
    kept = workspace_view(w, desc, params, "kept", torch.int32, (units, lay.kept_stride))[u, :ell].cpu().numpy()
    check_band(kept, O.pin_window(O.max_pool(s_ref, cfg.pool_kernel), T, cfg.w), ell, where)
    sel = O.select(O.pin_window(O.max_pool(S.astype(np.float64), cfg.pool_kernel), T, cfg.w), ell)
    np.testing.assert_array_equal(sel, kept, err_msg=where)
    # bytes: rank i of the unit holds the original row kept[i] (K and V) at (new_table[i // b], i % b)
    vt = v_rows(cfg, SEED, r, l, h, kept)
    tbl = w.tables[r].cpu().numpy()
    ranks = np.arange(ell)
    blk = torch.from_numpy(tbl[ranks // cfg.b].astype(np.int64)).to(w.k.device)
    slot = torch.from_numpy((ranks % cfg.b).astype(np.int64)).to(w.k.device)
    np.testing.assert_array_equal(w.k[l][blk, slot, h].cpu().numpy().view(np.uint16), kt[kept], err_msg=where)
    np.testing.assert_array_equal(w.v[l][blk, slot, h].cpu().numpy().view(np.uint16), vt, err_msg=where)
