"""Device-resident workloads: torch allocation + the Philox device generator (libzpcgen.so).

Input generation and memory plumbing only (no compression arithmetic). Used by tests, bench.py
and smoke(); it never imports the oracle.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from .workloads import Config, Layout, budgets_for, make_layout

HERE = os.path.dirname(os.path.abspath(__file__))
GEN_PATH = os.path.join(HERE, "lib", "libzpcgen.so")


class zpcgen_cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("L", "h_kv", "h_q", "d", "b", "N_total", "M", "w", "dtype",
                                               "structured", "prefix_tokens")] + [("seed", ctypes.c_uint64)]


_gen = None


def gen_lib():
    global _gen
    if _gen is None:
        if not os.path.exists(GEN_PATH):
            raise RuntimeError(f"{GEN_PATH} missing: run __graft_entry__.build()")
        g = ctypes.CDLL(GEN_PATH)
        g.zpcgen_fill_kv.argtypes = [ctypes.POINTER(zpcgen_cfg)] + [ctypes.c_void_p] * 3 + [ctypes.c_int32] + \
            [ctypes.c_void_p] * 2 + [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        g.zpcgen_fill_q.argtypes = [ctypes.POINTER(zpcgen_cfg)] + [ctypes.c_void_p] * 3 + [ctypes.c_int32,
                                                                                            ctypes.c_void_p]
        _gen = g
    return _gen


def storage_dtype(cfg: Config):
    return torch.float32 if cfg.dtype == "fp32" else torch.int16     # bf16 carried as raw 16-bit words


def to_dev(a: np.ndarray, device="cuda"):
    if a.dtype == np.uint16:
        a = a.view(np.int16)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def to_host(t: torch.Tensor, like_uint16=False):
    a = t.detach().cpu().numpy()
    return a.view(np.uint16) if like_uint16 else a


@dataclass
class DeviceWorkload:
    cfg: Config
    seed: int
    layout: Layout
    budgets_host: np.ndarray
    k: torch.Tensor
    v: torch.Tensor
    q: torch.Tensor
    q_slots: torch.Tensor
    seq_lens: torch.Tensor
    tables: torch.Tensor
    budgets: torch.Tensor
    new_lens: torch.Tensor
    new_num_blocks: torch.Tensor
    ref_counts: torch.Tensor | None
    free_stack: torch.Tensor
    free_top: torch.Tensor
    freed: torch.Tensor
    num_freed: torch.Tensor
    status: torch.Tensor
    workspace: torch.Tensor | None = None
    max_seq_len: int = 0
    f_cache: torch.Tensor | None = None          # NEXT-2 global-score pool
    is_compressed: torch.Tensor | None = None    # NEXT-2 [R]
    window_lse: torch.Tensor | None = None       # NEXT-4 fp32 [L][M][w][h_q] normalisers (ZPC_F_LSE_INPUT)


def alloc_outputs(R, L, h_kv, N_total, freed_capacity, device="cuda"):
    return dict(new_lens=torch.zeros((R, L, h_kv), dtype=torch.int32, device=device),
                new_num_blocks=torch.zeros(R, dtype=torch.int32, device=device),
                freed=torch.full((freed_capacity,), -1, dtype=torch.int32, device=device),
                num_freed=torch.zeros(1, dtype=torch.int32, device=device),
                status=torch.full((1,), 12345, dtype=torch.int32, device=device))


def freed_capacity_for(lay: Layout, cfg: Config) -> int:
    N = -(-lay.seq_lens // cfg.b)
    return int(max(1, (N - cfg.n_max).clip(min=0).sum() + lay.N_total))


def from_host(hw, device="cuda", max_seq_len=None) -> DeviceWorkload:
    """Copy a HostWorkload (zpc_inputs.make_host_workload) to the device."""
    cfg, lay = hw.cfg, hw.layout
    outs = alloc_outputs(len(lay.seq_lens), cfg.L, cfg.h_kv, lay.N_total, freed_capacity_for(lay, cfg), device)
    return DeviceWorkload(
        cfg=cfg, seed=hw.seed, layout=lay, budgets_host=hw.budgets,
        k=to_dev(hw.k_cache, device), v=to_dev(hw.v_cache, device), q=to_dev(hw.q_cache, device),
        q_slots=to_dev(lay.q_slots, device), seq_lens=to_dev(lay.seq_lens, device),
        tables=to_dev(lay.tables, device), budgets=to_dev(hw.budgets, device),
        ref_counts=None if lay.ref_counts is None else to_dev(lay.ref_counts, device),
        free_stack=to_dev(lay.free_stack, device),
        free_top=torch.tensor([lay.free_top], dtype=torch.int32, device=device),
        max_seq_len=int(max_seq_len or int(lay.seq_lens.max())),
        f_cache=None if getattr(hw, "f_cache", None) is None else to_dev(hw.f_cache, device),
        is_compressed=None if getattr(hw, "is_compressed", None) is None else to_dev(hw.is_compressed, device),
        **outs)


def generate(cfg: Config, seed: int, rids, device="cuda", table_stride=None) -> DeviceWorkload:
    """Full-size workload generated directly in HBM by the Philox device twin."""
    lay = make_layout(cfg, seed, rids, table_stride)
    R = len(lay.seq_lens)
    sdt = storage_dtype(cfg)
    k = torch.zeros((cfg.L, lay.N_total, cfg.b, cfg.h_kv, cfg.d), dtype=sdt, device=device)
    v = torch.zeros_like(k)
    q = torch.zeros((cfg.L, lay.M, cfg.w, cfg.h_q, cfg.d), dtype=sdt, device=device)
    bud = budgets_for(cfg, seed, lay.rids)
    outs = alloc_outputs(R, cfg.L, cfg.h_kv, lay.N_total, freed_capacity_for(lay, cfg), device)
    dw = DeviceWorkload(
        cfg=cfg, seed=seed, layout=lay, budgets_host=bud, k=k, v=v, q=q,
        q_slots=to_dev(lay.q_slots, device), seq_lens=to_dev(lay.seq_lens, device),
        tables=to_dev(lay.tables, device), budgets=to_dev(bud, device),
        ref_counts=None if lay.ref_counts is None else to_dev(lay.ref_counts, device),
        free_stack=to_dev(lay.free_stack, device),
        free_top=torch.tensor([lay.free_top], dtype=torch.int32, device=device),
        max_seq_len=int(lay.seq_lens.max()), **outs)
    gc = zpcgen_cfg(cfg.L, cfg.h_kv, cfg.h_q, cfg.d, cfg.b, lay.N_total, lay.M, cfg.w,
                    0 if cfg.dtype == "bf16" else 1, int(cfg.structured), cfg.prefix_tokens, seed)
    rids_d = torch.from_numpy(lay.rids.astype(np.int32)).to(device)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    g = gen_lib()
    rc = g.zpcgen_fill_kv(ctypes.byref(gc), ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()),
                          ctypes.c_void_p(dw.tables.data_ptr()), lay.table_stride,
                          ctypes.c_void_p(dw.seq_lens.data_ptr()), ctypes.c_void_p(rids_d.data_ptr()), R,
                          int(lay.seq_lens.max()), stream)
    assert rc == 0
    rc = g.zpcgen_fill_q(ctypes.byref(gc), ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(dw.q_slots.data_ptr()),
                         ctypes.c_void_p(rids_d.data_ptr()), R, stream)
    assert rc == 0
    torch.cuda.synchronize()
    return dw
