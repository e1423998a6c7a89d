"""Convenience glue: build the C structs for a set of device tensors and call the ABI.

Duck-typed over any object with the DeviceWorkload attributes (cfg, layout, k, v, q, q_slots,
seq_lens, tables, budgets, new_lens, new_num_blocks, ref_counts, free_stack, free_top, freed,
num_freed, status, workspace, max_seq_len). Marshalling only.
"""
from __future__ import annotations

import torch

from . import zipc


def desc_params(w, flags=0, pool_kernel=None, max_seq_len=None, redundancy=None, global_alpha=None,
                lse_input=False):
    """redundancy: None, or (lambda, tau, p) -> sets ZPC_F_REDUNDANCY with those parameters.
    global_alpha: None, or alpha -> sets ZPC_F_GLOBAL_SCORE (w.f_cache / w.is_compressed must exist).
    lse_input: sets ZPC_F_LSE_INPUT (w.window_lse must exist: fp32 [L][M][w][h_q])."""
    cfg, lay = w.cfg, w.layout
    desc = zipc.make_desc(cfg.L, cfg.h_kv, cfg.h_q, cfg.d, cfg.b, lay.N_total, lay.M, cfg.w, cfg.dtype)
    if w.ref_counts is not None:
        flags |= zipc.ZPC_F_PREFIX
    extra = {}
    if global_alpha is not None:
        flags |= zipc.ZPC_F_GLOBAL_SCORE
        extra["global_alpha"] = global_alpha
    if lse_input:
        flags |= zipc.ZPC_F_LSE_INPUT
    if redundancy is not None:
        flags |= zipc.ZPC_F_REDUNDANCY
        extra.update(redundancy_lambda=redundancy[0], redundancy_tau=redundancy[1], redundancy_p=redundancy[2])
    params = zipc.make_params(cfg.n_max, cfg.pool_kernel if pool_kernel is None else pool_kernel,
                              int(max_seq_len or w.max_seq_len), flags, **extra)
    return desc, params


def ensure_workspace(w, desc, params):
    need = zipc.zpc_workspace_bytes(desc, params, int(w.seq_lens.numel()))
    if need == 0:
        raise zipc.ZipcError(zipc.ZPC_ERR_INVALID_ARG, "zpc_workspace_bytes")
    if w.workspace is None or w.workspace.numel() < need:
        w.workspace = torch.empty(need, dtype=torch.uint8, device=w.k.device)
    return w.workspace


def batch_of(w, desc, params):
    ensure_workspace(w, desc, params)
    return zipc.make_batch(k_cache=w.k, v_cache=w.v, q_cache=w.q, q_slots=w.q_slots, seq_lens=w.seq_lens,
                           block_tables=w.tables, budgets=w.budgets, new_lens=w.new_lens,
                           new_num_blocks=w.new_num_blocks, ref_counts=w.ref_counts, free_stack=w.free_stack,
                           free_top=w.free_top, freed_blocks=w.freed, num_freed=w.num_freed,
                           workspace=w.workspace, status=w.status,
                           global_scores=getattr(w, "f_cache", None), is_compressed=getattr(w, "is_compressed", None),
                           window_lse=getattr(w, "window_lse", None))


def workspace_view(w, desc, params, name, dtype, shape):
    """A typed view of one workspace region (scores, kept, targets, ...) for inspection."""
    lay = zipc.zpc_workspace_layout_get(desc, params, int(w.seq_lens.numel()))
    off = getattr(lay, name)
    n = 1
    for s in shape:
        n *= s
    esz = torch.tensor([], dtype=dtype).element_size()
    return w.workspace[off:off + n * esz].view(dtype).view(*shape)
