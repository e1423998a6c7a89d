"""Synthetic workloads shaped like BASELINE.json's configs (recipe: DESIGN.md §Inputs).

Everything here is integer arithmetic until the final exact scaling by 2^-15 and
the round-to-nearest-even to bf16, so the device twin (csrc/zpc_gen.cu) produces
bit-identical bytes. Rows are keyed by LOGICAL identity (request id, layer, head,
position), never by physical block, so a request's data does not depend on its
block placement or on which GPU it is sharded to.

Element recipe (d elements per row, element pair i from one Philox call):
  z        = u0+u1+u2+u3 - 2*65535         (Irwin-Hall(4) of 16-bit uniforms, std ~37838)
  dir[l,h] = +-1 per element               (fixed per layer, KV head)
  K        = (z + A_t * dir) * 2^-15       A_t in units of 8192: sink (t<4) 6, heavy hitter
                                           (p=5/256) 3..5, recency (last 256 tokens) >= 2
  V        = z * 2^-15
  Q (u,hq) = (z + 2*8192 * dir[l, hq//G]) * 2^-15
"""
from __future__ import annotations

from dataclasses import dataclass, field

import math

import numpy as np

from .philox import philox4x32

KIND_K, KIND_V, KIND_Q, KIND_DIR, KIND_ROLE, KIND_BUDGET, KIND_PERM = 1, 2, 3, 4, 5, 6, 7
PREFIX_RID = 0xFFFFFF  # request id used to key shared-prefix tokens
AMP_UNIT = 8192
Q_AMP = 2 * AMP_UNIT
SINKS = 4
RECENT = 256


@dataclass
class Config:
    name: str
    L: int
    h_kv: int
    h_q: int
    d: int
    b: int
    dtype: str
    w: int
    n_max: int
    pool_kernel: int
    seq_lens: list            # per request (global ids)
    budget: int | tuple       # int = uniform, (lo, hi) = per-head U{lo..hi}
    prefix_tokens: int = 0    # shared prefix length (multiple of b) for config 5
    wave: int = 0             # requests per wave per GPU (0 = all)
    free_slack: int = 64      # extra free blocks beyond fresh demand
    structured: bool = True
    notes: str = ""

    @property
    def G(self):
        return self.h_q // self.h_kv

    @property
    def R(self):
        return len(self.seq_lens)


def _cfgs():
    return {
        # BASELINE.json configs[0]: Figure-1 toy (h_q = 4 is our proposal, G = 2)
        "toy": Config("toy", L=1, h_kv=2, h_q=4, d=64, b=4, dtype="fp32", w=2, n_max=4,
                      pool_kernel=1, seq_lens=[20, 25], budget=12, free_slack=4),
        # configs[1]: Qwen2.5-7B-shaped (h_q = 28 from the public model config)
        "qwen7b": Config("qwen7b", L=28, h_kv=4, h_q=28, d=128, b=16, dtype="bf16", w=32, n_max=129,
                         pool_kernel=7, seq_lens=[8192] * 64, budget=2048),
        # configs[2]: Llama-3.1-8B-shaped, mixed per-head budgets
        "llama8b": Config("llama8b", L=32, h_kv=8, h_q=32, d=128, b=16, dtype="bf16", w=32, n_max=129,
                          pool_kernel=7, seq_lens=[16384] * 256, budget=(32, 2048), wave=32),
        # configs[3]: Qwen2.5-32B-shaped
        "qwen32b": Config("qwen32b", L=64, h_kv=8, h_q=40, d=128, b=16, dtype="bf16", w=32, n_max=129,
                          pool_kernel=7, seq_lens=[32768] * 512, budget=2048, wave=16),
        # configs[4]: shared prefix, 7B shape (proposal)
        "prefix": Config("prefix", L=28, h_kv=4, h_q=28, d=128, b=16, dtype="bf16", w=32, n_max=129,
                         pool_kernel=7, seq_lens=[4096 + 8192] * 1024, budget=2048, prefix_tokens=4096,
                         wave=128),
        # NEXT-3: the paper's operating point (b = 256, w = 16; budget 2048 -> N_max = 9),
        # Qwen3-8B shape (L = 36, h_kv = 8, h_q = 32, d = 128 from the public model config), steady
        # state T = N_max * b (exactly one block evicted per call), ~1/b of the running requests per call
        # (PAPER.md:153): 4 requests per call per GPU
        "paper_op": Config("paper_op", L=36, h_kv=8, h_q=32, d=128, b=256, dtype="bf16", w=16, n_max=9,
                           pool_kernel=7, seq_lens=[2304] * 64, budget=2048, wave=4, free_slack=4),
    }


CONFIGS = _cfgs()


def scaled(cfg: Config, **kw) -> Config:
    """A copy of cfg with fields replaced (used for small parity cases of a config's shape)."""
    d = dict(cfg.__dict__)
    d.update(kw)
    return Config(**d)


# ------------------------------------------------------------------ elements
def _kindword(kind, l, h):
    return np.uint32((kind << 24) | (l << 8) | h)


def irwin_hall_rows(kind, seed, rid, l, head, pos, d):
    """z integers [len(pos), d] for rows keyed by (kind, rid, l, head, pos)."""
    pos = np.asarray(pos, dtype=np.uint32)
    i = np.arange(d // 2, dtype=np.uint32)
    x0, x1, x2, x3 = philox4x32(pos[:, None], np.uint32(rid), _kindword(kind, l, head), i[None, :],
                                seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    m = np.uint32(0xFFFF)
    za = ((x0 & m).astype(np.int64) + (x0 >> 16) + (x1 & m) + (x1 >> 16)) - 2 * 65535
    zb = ((x2 & m).astype(np.int64) + (x2 >> 16) + (x3 & m) + (x3 >> 16)) - 2 * 65535
    z = np.empty((len(pos), d), np.int64)
    z[:, 0::2] = za
    z[:, 1::2] = zb
    return z


def direction(seed, l, h, d):
    i = np.arange(d, dtype=np.uint32)
    x0, _, _, _ = philox4x32(i, np.uint32(0), _kindword(KIND_DIR, l, h), np.uint32(0),
                             seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    return np.where((x0 & 1) == 1, 1, -1).astype(np.int64)


def token_amp(seed, rid, l, h, pos, T, structured=True):
    """A_t in units of AMP_UNIT for key rows (sinks, heavy hitters, recency)."""
    pos = np.asarray(pos, dtype=np.int64)
    if not structured:
        return np.zeros(len(pos), np.int64)
    x0, _, _, _ = philox4x32(pos.astype(np.uint32), np.uint32(rid), _kindword(KIND_ROLE, l, h), np.uint32(0),
                             seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    heavy = (x0 & 0xFF) < 5
    cat = (x0 >> 8) & 3
    amp = np.where(heavy, np.array([3, 4, 5, 4], np.int64)[cat], 0)
    amp = np.where(pos < SINKS, 6, amp)
    amp = np.where(pos >= T - RECENT, np.maximum(amp, 2), amp)
    return amp


def to_storage(x_int: np.ndarray, dtype: str) -> np.ndarray:
    """Exact x_int * 2^-15 in fp32, then RNE to bf16 bits (or keep fp32)."""
    f = (x_int.astype(np.float64) * (2.0 ** -15)).astype(np.float32)   # exact: |x_int| < 2^24
    if dtype == "fp32":
        return f
    bits = f.view(np.uint32).astype(np.uint64)
    rounded = (bits + 0x7FFF + ((bits >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def k_rows(cfg: Config, seed, rid, l, h, pos, T):
    pos = np.asarray(pos)
    rid_arr = np.where(pos < cfg.prefix_tokens, PREFIX_RID, rid)
    out = np.empty((len(pos), cfg.d), np.int64)
    dirv = direction(seed, l, h, cfg.d)
    for key in np.unique(rid_arr):
        sel = rid_arr == key
        z = irwin_hall_rows(KIND_K, seed, int(key), l, h, pos[sel], cfg.d)
        # recency is relative to the request's own length; prefix tokens are never recent
        amp = token_amp(seed, int(key), l, h, pos[sel], T, cfg.structured)
        out[sel] = z + (amp * AMP_UNIT)[:, None] * dirv[None, :]
    return to_storage(out, cfg.dtype)


def v_rows(cfg: Config, seed, rid, l, h, pos):
    pos = np.asarray(pos)
    rid_arr = np.where(pos < cfg.prefix_tokens, PREFIX_RID, rid)
    out = np.empty((len(pos), cfg.d), np.int64)
    for key in np.unique(rid_arr):
        sel = rid_arr == key
        out[sel] = irwin_hall_rows(KIND_V, seed, int(key), l, h, pos[sel], cfg.d)
    return to_storage(out, cfg.dtype)


def q_rows(cfg: Config, seed, rid, l):
    """Window queries of one request and layer: [w, h_q, d] storage elements."""
    out = np.empty((cfg.w, cfg.h_q, cfg.d), np.int64)
    for hq in range(cfg.h_q):
        z = irwin_hall_rows(KIND_Q, seed, rid, l, hq, np.arange(cfg.w), cfg.d)
        amp = Q_AMP if cfg.structured else 0
        out[:, hq, :] = z + amp * direction(seed, l, hq // cfg.G, cfg.d)[None, :]
    return to_storage(out, cfg.dtype)


def budgets_for(cfg: Config, seed, rids):
    R = len(rids)
    if isinstance(cfg.budget, int):
        return np.full((R, cfg.L, cfg.h_kv), cfg.budget, np.int32)
    lo, hi = cfg.budget
    out = np.empty((R, cfg.L, cfg.h_kv), np.int32)
    for i, rid in enumerate(rids):
        for l in range(cfg.L):
            x0, _, _, _ = philox4x32(np.arange(cfg.h_kv, dtype=np.uint32), np.uint32(rid),
                                     _kindword(KIND_BUDGET, l, 0), np.uint32(0),
                                     seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
            out[i, l] = lo + (x0 % np.uint32(hi - lo + 1)).astype(np.int32)
    return out


# ------------------------------------------------------------------ layout
@dataclass
class Layout:
    """Block bookkeeping of one shard (the requests one GPU compresses in one wave)."""
    rids: np.ndarray
    seq_lens: np.ndarray
    tables: np.ndarray
    table_stride: int
    q_slots: np.ndarray
    M: int
    N_total: int
    free_stack: np.ndarray
    free_top: int
    ref_counts: np.ndarray | None
    prefix_blocks: np.ndarray = field(default=None)


def make_layout(cfg: Config, seed, rids, table_stride=None) -> Layout:
    """Fragmented tables: a seeded permutation of the shard's pool."""
    rids = np.asarray(rids, np.int64)
    R = len(rids)
    T = np.array([cfg.seq_lens[r] for r in rids], np.int32)
    N = -(-T // cfg.b)
    n_pref = cfg.prefix_tokens // cfg.b
    priv = N - n_pref
    nm1 = cfg.n_max - 1
    fresh_demand = R * (min(n_pref, nm1) + (1 if max(n_pref, nm1) >= N.min() else 0)) if n_pref else 0
    N_total = int(n_pref + priv.sum() + fresh_demand + cfg.free_slack)
    x0, x1, _, _ = philox4x32(np.arange(N_total, dtype=np.uint32), np.uint32(len(rids)),
                              np.uint32(KIND_PERM << 24), np.uint32(int(rids[0]) if R else 0),
                              seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    keys = (x0.astype(np.uint64) << np.uint64(32)) | x1.astype(np.uint64)
    perm = np.argsort(keys, kind="stable").astype(np.int32)
    stride = int(table_stride or N.max())
    tables = np.full((R, stride), -1, np.int32)
    cur = 0
    prefix = perm[:n_pref].copy()
    cur = n_pref
    for i in range(R):
        tables[i, :n_pref] = prefix
        tables[i, n_pref:N[i]] = perm[cur:cur + priv[i]]
        cur += int(priv[i])
    free = perm[cur:].copy()
    stack = np.zeros(N_total, np.int32)
    stack[:len(free)] = free
    refs = None
    if n_pref:
        refs = np.zeros(N_total, np.int32)
        refs[tables[tables >= 0]] = 1
        refs[prefix] = R + 1          # every request + the harness's own reference
    M = R + 3
    # distinct, non-identity slots: stride coprime to M (a permutation of the M slots)
    stride_q = next(s for s in range(5, 5 + M + 1) if math.gcd(s, M) == 1)
    q_slots = ((np.arange(R) * stride_q + 2) % M).astype(np.int32)
    return Layout(rids=rids, seq_lens=T, tables=tables, table_stride=stride, q_slots=q_slots, M=M,
                  N_total=N_total, free_stack=stack, free_top=len(free), ref_counts=refs,
                  prefix_blocks=prefix)


@dataclass
class HostWorkload:
    cfg: Config
    seed: int
    layout: Layout
    budgets: np.ndarray
    k_cache: np.ndarray
    v_cache: np.ndarray
    q_cache: np.ndarray
    f_cache: np.ndarray | None = None        # NEXT-2 global-score pool (global_history)
    is_compressed: np.ndarray | None = None  # NEXT-2 [R]


def make_host_workload(cfg: Config, seed: int, rids=None, table_stride=None) -> HostWorkload:
    """Fully materialised host arrays (small configs / parity cases only)."""
    rids = np.arange(cfg.R) if rids is None else np.asarray(rids)
    lay = make_layout(cfg, seed, rids, table_stride)
    sdt = np.float32 if cfg.dtype == "fp32" else np.uint16
    K = np.zeros((cfg.L, lay.N_total, cfg.b, cfg.h_kv, cfg.d), sdt)
    V = np.zeros_like(K)
    Q = np.zeros((cfg.L, lay.M, cfg.w, cfg.h_q, cfg.d), sdt)
    for i, rid in enumerate(lay.rids):
        T = int(lay.seq_lens[i])
        t = np.arange(T)
        blk = lay.tables[i, t // cfg.b]
        for l in range(cfg.L):
            for h in range(cfg.h_kv):
                K[l, blk, t % cfg.b, h] = k_rows(cfg, seed, int(rid), l, h, t, T)
                V[l, blk, t % cfg.b, h] = v_rows(cfg, seed, int(rid), l, h, t)
            Q[l, lay.q_slots[i]] = q_rows(cfg, seed, int(rid), l)
    return HostWorkload(cfg=cfg, seed=seed, layout=lay, budgets=budgets_for(cfg, seed, lay.rids),
                        k_cache=K, v_cache=V, q_cache=Q)


# ------------------------------------------------------------------ NEXT-2 inputs (random numbers only)
KIND_GLOBAL = 9


def global_history(cfg: Config, seed, N_total: int, rids, scale=None):
    """Previous global scores F [L, N_total, b, h_kv] fp32 (Philox uniform in [0, scale); scale ~ the
    mean attention score 2/T) and is_compressed [R] int32 (every even global request id has been
    compressed before). Seeded random inputs, no method arithmetic."""
    rids = np.asarray(rids)
    if scale is None:
        scale = 2.0 / float(np.mean([cfg.seq_lens[int(r)] for r in rids]))
    n = cfg.L * N_total * cfg.b * cfg.h_kv
    x0, _, _, _ = philox4x32(np.arange(n, dtype=np.uint32), np.uint32(0), np.uint32(KIND_GLOBAL << 24),
                             np.uint32(0), seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    f = ((x0 >> 8).astype(np.float64) * (1.0 / (1 << 24)) * scale).astype(np.float32)
    comp = (rids % 2 == 0).astype(np.int32)
    return f.reshape(cfg.L, N_total, cfg.b, cfg.h_kv), comp
