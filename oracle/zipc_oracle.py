"""fp64 CPU oracle of the Zipage compression step (TEST INFRASTRUCTURE ONLY).

Every function cites the passage of /root/reference/PAPER.md (arXiv 2603.08743)
it follows, as ``PAPER.md:<line> (<section / Alg / Eq>)``. Where the paper is
silent or garbled, the reading taken is the numbered one of SURVEY.md §8(c),
restated in DESIGN.md §Readings as R1..R17.

Data conventions (plain numpy; nothing here imports the CUDA product):
  * K, V pools: arrays [L, N_total, b, h_kv, d] of raw element bits —
    ``np.uint16`` for bf16 (bf16 bits), ``np.float32`` for fp32.
  * Q window cache: [L, M, w, h_q, d], same element type; row u of slot j is
    the query of position T-w+u (R3).
  * block tables: int32 [R, stride]; seq_lens int32 [R]; budgets int32 [R, L, h_kv].
  * free stack: int32 [capacity] with valid entries [0, top); pop takes
    stack[top-1].
All floating-point arithmetic is fp64 on exactly-widened inputs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Status codes (same numeric values the C-ABI documents; restated here, not
# imported, so that the oracle shares nothing with the product).
OK = 0
ERR_NOT_TRIGGERED = -10
ERR_BAD_TABLE = -11
ERR_BAD_BUDGET = -12
ERR_NO_FREE_BLOCKS = -13
ERR_SEQ_TOO_LONG = -14
ERR_BAD_SLOT = -15
ERR_CAPACITY = -16
ERR_NONFINITE = -17   # F_VALIDATE: a Q or K element the call reads is Inf/NaN (ABI-level check, R33)

F_PREFIX = 1
F_VALIDATE = 2
F_REDUNDANCY = 16   # NEXT-1: lightning redundancy + temperature softmax + S - lambda*R
F_GLOBAL_SCORE = 32  # NEXT-2: global score (Alg. 2) + F relocation with the kept rows
F_POOL_FIRST = 128   # pool (MaxPool1D) only at a request's first compression (R32)


@dataclass
class Geometry:
    """Pool geometry, PAPER.md:42 (§3 'Pre-allocated memory') and :69 (§4.2, Q cache)."""
    L: int
    h_kv: int
    h_q: int
    d: int
    b: int
    N_total: int
    M: int
    w: int
    dtype: str  # "bf16" | "fp32"

    @property
    def G(self) -> int:
        return self.h_q // self.h_kv


@dataclass
class Params:
    n_max: int
    pool_kernel: int = 1
    max_seq_len: int = 1 << 30
    flags: int = 0
    lam: float = 0.2      # lambda, PAPER.md:718 (§C.8 recommended)
    tau: float = 0.4      # tau
    sim_p: float = 0.8    # similarity threshold p: no value in the paper (R19)
    alpha: float = 0.8    # global-score decay, PAPER.md:718 (§C.8 recommended)


# --------------------------------------------------------------------------
# element widening (exact)
# --------------------------------------------------------------------------
def widen(x: np.ndarray, dtype: str) -> np.ndarray:
    """Exact widening of stored elements to fp64. bf16 bits -> fp32 -> fp64 is exact."""
    if dtype == "bf16":
        return (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    if dtype == "fp32":
        return x.astype(np.float64)
    raise ValueError(dtype)


# --------------------------------------------------------------------------
# a0: validate and plan targets — PAPER.md:61-66 (§4.1), :131-138 (§4.5)
# --------------------------------------------------------------------------
@dataclass
class Plan:
    status: int
    n_blocks: np.ndarray = field(default=None)   # N per request
    n_prefix: np.ndarray = field(default=None)   # shared leading blocks (R11)
    targets: np.ndarray = field(default=None)    # [R, n_max-1] physical ids
    reserved: np.ndarray = field(default=None)   # [R]
    fresh: list = field(default=None)            # per request: fresh ids in pop order


def _request_error(geo, prm, r, seq_lens, tables, table_stride, budgets, ref_counts, q_slots):
    """Per-request checks in the fixed order of DESIGN.md §Errors. Returns (err, N, n_prefix)."""
    T = int(seq_lens[r])
    if q_slots is not None and not (0 <= int(q_slots[r]) < geo.M):
        return ERR_BAD_SLOT, 0, 0
    if T > prm.max_seq_len:
        return ERR_SEQ_TOO_LONG, 0, 0
    N = -(-T // geo.b)  # ceil(T/b): blocks occupied
    if N > table_stride:
        return ERR_BAD_TABLE, N, 0
    # trigger: N >= N_max (R14 allows a partial last block)
    if N < prm.n_max:
        return ERR_NOT_TRIGGERED, N, 0
    row = [int(x) for x in tables[r, :N]]
    if any(bid < 0 or bid >= geo.N_total for bid in row):
        return ERR_BAD_TABLE, N, 0
    if (prm.flags & F_VALIDATE) and len(set(row)) != len(row):
        return ERR_BAD_TABLE, N, 0
    n_prefix = 0
    if prm.flags & F_PREFIX:
        # shared = reference count > 1; R11: must be a leading run
        while n_prefix < N and ref_counts[row[n_prefix]] > 1:
            n_prefix += 1
        if any(ref_counts[bid] > 1 for bid in row[n_prefix:]):
            return ERR_BAD_TABLE, N, n_prefix
    kmax = (prm.n_max - 1) * geo.b  # k = (N_max-1)*b
    bud = budgets[r]
    if np.any(bud < geo.w) or np.any(bud > kmax):
        return ERR_BAD_BUDGET, N, n_prefix
    return OK, N, n_prefix


def plan(geo: Geometry, prm: Params, seq_lens, tables, budgets, ref_counts=None,
         free_stack=None, free_top=0, q_slots=None, free_capacity=None, freed_capacity=None) -> Plan:
    """Trigger check, prefix-aware target choice (§4.5 bullets), fresh pops.

    Targets (R9, R10): N_prefix = 0 -> own table[0..N_max-2] (Fig. 1: "moved to the
    first three blocks"). N_prefix >= N_max-1 -> N_max-1 fresh blocks
    (PAPER.md:134). Otherwise fresh for j < N_prefix, own table[j] for j >= N_prefix
    (PAPER.md:135). Reserved = own table[max(N_prefix, N_max-1)], or one more fresh
    pop when the table is wholly shared. Fresh blocks pop from the free-stack top
    in (request, target index) order, the reserved pop last.
    """
    R = len(seq_lens)
    table_stride = tables.shape[1] if R else 0
    nb = np.zeros(R, np.int64)
    npf = np.zeros(R, np.int64)
    for r in range(R):
        err, N, n_prefix = _request_error(geo, prm, r, seq_lens, tables, table_stride,
                                          budgets, ref_counts, q_slots)
        if err != OK:
            return Plan(status=err)
        nb[r], npf[r] = N, n_prefix
    nm1 = prm.n_max - 1
    targets = np.zeros((R, nm1), np.int32)
    reserved = np.zeros(R, np.int32)
    fresh_lists = []
    top = int(free_top)
    # demand check before any pop (all-or-nothing)
    demand = 0
    for r in range(R):
        n_fresh = min(int(npf[r]), nm1)
        res_idx = max(int(npf[r]), nm1)
        demand += n_fresh + (1 if res_idx >= nb[r] else 0)
    if demand > top:
        return Plan(status=ERR_NO_FREE_BLOCKS)
    if freed_capacity is not None or free_capacity is not None:
        # R18: capacity is checked against exactly the blocks the call will free — private
        # non-target blocks plus shared blocks whose every reference is held by this batch.
        priv = sum(max(0, int(nb[r]) - 1 - max(int(npf[r]), nm1)) for r in range(R))
        occ = {}
        for r in range(R):
            for j in range(int(npf[r])):
                occ[int(tables[r, j])] = occ.get(int(tables[r, j]), 0) + 1
        zeroed = sum(1 for bid, n in occ.items() if n == ref_counts[bid])
        if freed_capacity is not None and priv + zeroed > freed_capacity:
            return Plan(status=ERR_CAPACITY)
        if free_capacity is not None and top - demand + priv + zeroed > free_capacity:
            return Plan(status=ERR_CAPACITY)
    for r in range(R):
        N, n_prefix = int(nb[r]), int(npf[r])
        row = tables[r]
        fr = []
        for j in range(nm1):
            if j < n_prefix:  # fresh target (j < min(N_prefix, N_max-1))
                top -= 1
                targets[r, j] = free_stack[top]
                fr.append(int(targets[r, j]))
            else:             # reuse own block at the same logical index
                targets[r, j] = row[j]
        res_idx = max(n_prefix, nm1)
        if res_idx < N:
            reserved[r] = row[res_idx]
        else:
            top -= 1
            reserved[r] = free_stack[top]
            fr.append(int(reserved[r]))
        fresh_lists.append(fr)
    return Plan(status=OK, n_blocks=nb, n_prefix=npf, targets=targets, reserved=reserved,
                fresh=fresh_lists)


# --------------------------------------------------------------------------
# a1: window-query x key logits — Alg. 1, PAPER.md:369-405 (§C.2)
# --------------------------------------------------------------------------
def _group(geo: Geometry, h: int):
    """R5: query head i uses KV head floor(i/G) -> group of KV head h = [h*G, h*G+G)."""
    return range(h * geo.G, (h + 1) * geo.G)


def logits_blockwise(geo: Geometry, q_slot_l: np.ndarray, k_layer: np.ndarray, table, T: int, h: int,
                     ) -> np.ndarray:
    """Formulation A: Alg. 1 block by block.

    q_slot_l: [w, h_q, d] fp64 (one layer, one query slot); k_layer: [N_total, b, h_kv, d] fp64.
    Returns A: [G, w, N*b] fp64 with -inf at masked / out-of-sequence entries.
    A'[u, v] = Q_j K_i^T / sqrt(d). Mask (R1, R2): window row u is
    position p_u = T-w+u; entry t is masked iff t > p_u; slots t >= T are not tokens.
    """
    w, b, d = geo.w, geo.b, geo.d
    N = -(-T // b)
    out = np.full((geo.G, w, N * b), -np.inf)
    for gi, g in enumerate(_group(geo, h)):
        Qj = q_slot_l[:, g, :]                       # [w, d]  (Alg.1 line 2)
        for i in range(N):                           # parallel over blocks
            Ki = k_layer[table[i], :, h, :]          # [b, d]  (Alg.1 lines 3-5)
            Ap = (Qj @ Ki.T) / math.sqrt(d)          # [w, b]  (Alg.1 line 6)
            for u in range(w):
                for v in range(b):
                    t = i * b + v
                    if t >= T or t > T - w + u:
                        Ap[u, v] = -np.inf
            out[gi, :, i * b:(i + 1) * b] = Ap       # A[i] <- A' (Alg.1 line 11)
    return out


def logits_dense(geo: Geometry, q_slot_l: np.ndarray, k_layer: np.ndarray, table, T: int, h: int
                 ) -> np.ndarray:
    """Formulation B: gather K densely into [T, d], one matrix product per query head.
    Returns [G, w, T] with -inf where t > T-w+u."""
    b = geo.b
    t = np.arange(T)
    Kd = k_layer[np.asarray(table)[t // b], t % b, h, :]       # [T, d]
    out = np.empty((geo.G, geo.w, T))
    for gi, g in enumerate(_group(geo, h)):
        out[gi] = (q_slot_l[:, g, :] @ Kd.T) / math.sqrt(geo.d)
    u = np.arange(geo.w)[:, None]
    mask = t[None, :] > (T - geo.w + u)
    out[:, mask] = -np.inf
    return out


# --------------------------------------------------------------------------
# a2: softmax over the window row, GQA max, mean over window — PAPER.md:409-411
# --------------------------------------------------------------------------
def attention_scores(A: np.ndarray, T: int) -> np.ndarray:
    """A: [G, w, >=T] logits with -inf masks. Reshape to w x (N b) and softmax along
    the last dim, max-reduce over the query heads of the KV group,
    then mean over the w window rows. Returns s: [T] fp64."""
    A = A[:, :, :T]
    m = A.max(axis=2, keepdims=True)
    E = np.exp(A - m)                      # exp(-inf) = 0 for masked entries
    P = E / E.sum(axis=2, keepdims=True)   # softmax per (g, u)
    return P.max(axis=0).mean(axis=0)      # max over g, then mean over u


# --------------------------------------------------------------------------
# NEXT-4: single-pass scoring with the window normalisers given (derived from
# PAPER.md:409-411). The softmax of window row u is exp(A[g,u,t] - LSE[g,u]) with
# LSE[g,u] = log sum_{t <= T-w+u} exp(A[g,u,t]); decode attention of position T-w+u attends over exactly
# the keys 0..T-w+u with the same 1/sqrt(d) logits, so a serving engine already holds LSE.
# --------------------------------------------------------------------------
def window_lse(A: np.ndarray, T: int) -> np.ndarray:
    """LSE[g, u] = log sum_t exp(A[g, u, t]) over the unmasked entries (natural log), A as in
    attention_scores. The normaliser of PAPER.md:409's softmax, written out."""
    A = A[:, :, :T]
    m = A.max(axis=2)
    return m + np.log(np.exp(A - m[:, :, None]).sum(axis=2))


def attention_scores_given_lse(A: np.ndarray, lse: np.ndarray, T: int) -> np.ndarray:
    """s[t] = (1/w) sum_u max_g exp(A[g,u,t] - lse[g,u]) (PAPER.md:409-411 with the softmax normaliser
    supplied instead of recomputed). Equals attention_scores(A, T) when lse = window_lse(A, T)."""
    P = np.exp(A[:, :, :T] - lse[:, :, None])    # masked entries: exp(-inf) = 0
    return P.max(axis=0).mean(axis=0)


def unit_window_lse(geo: Geometry, window_lse_in: np.ndarray, slot: int, l: int, h: int) -> np.ndarray:
    """[G, w] slice of a window_lse array laid out [L][M][w][h_q] (the ABI's layout), group of KV head h
    (R5)."""
    return np.asarray(window_lse_in[l, slot][:, list(_group(geo, h))], np.float64).T


def unit_scores(geo: Geometry, q_cache_f64, k_pool_f64, table, T: int, slot: int, l: int, h: int,
                blockwise: bool = False, window_lse_in=None) -> np.ndarray:
    """S for one unit (request, layer, KV head) from widened caches; with window_lse_in
    ([L][M][w][h_q]) the normalisers are taken from it (NEXT-4)."""
    q = q_cache_f64[l, slot]           # [w, h_q, d]
    kl = k_pool_f64[l]                 # [N_total, b, h_kv, d]
    A = (logits_blockwise if blockwise else logits_dense)(geo, q, kl, table, T, h)
    if window_lse_in is not None:
        return attention_scores_given_lse(A, unit_window_lse(geo, window_lse_in, slot, l, h), T)
    return attention_scores(A, T)


def all_window_lse(geo: Geometry, q_cache, k_cache, q_slots, seq_lens, tables) -> np.ndarray:
    """The [L][M][w][h_q] normaliser array a decode engine would hold for these requests (slots not
    bound to a request stay 0): window_lse of every unit, by definition."""
    out = np.zeros((geo.L, geo.M, geo.w, geo.h_q))
    qf, kf = widen(q_cache, geo.dtype), widen(k_cache, geo.dtype)
    for r in range(len(seq_lens)):
        T, slot = int(seq_lens[r]), int(q_slots[r])
        for l in range(geo.L):
            for h in range(geo.h_kv):
                A = logits_dense(geo, qf[l, slot], kf[l], tables[r], T, h)
                out[l, slot][:, list(_group(geo, h))] = window_lse(A, T).T
    return out


# --------------------------------------------------------------------------
# a3: MaxPool1D and window pin — PAPER.md:480-487 (§C.4), :85, :591
# --------------------------------------------------------------------------
def max_pool(s: np.ndarray, k: int) -> np.ndarray:
    """S = MaxPool1D(S); R6: odd kernel, stride 1, same length,
    out-of-range neighbours ignored."""
    if k == 1:
        return s.copy()
    r = k // 2
    T = len(s)
    return np.array([s[max(0, t - r):min(T, t + r + 1)].max() for t in range(T)])


def pin_window(s: np.ndarray, T: int, w: int) -> np.ndarray:
    """Entries of the observation window get +inf."""
    out = s.copy()
    out[T - w:T] = np.inf
    return out


# --------------------------------------------------------------------------
# NEXT-1: lightning redundancy, temperature softmax, S - lambda*R
#   PAPER.md:498-507 (§C.5, redundancy score + Eq. S = S - lambda R), :616-620 (§C.7 lightning
#   redundancy: similarity only between keys of the same block), :677 (§C.8 temperature tau)
# Readings: R19 p is a parameter (no value in the paper); R20 "normalized by the
# sequence length" divides by T and slots >= T take no part; R21 "exceeding" is strictly greater,
# the diagonal is zeroed first, "last" is the largest row index (newest token); R22 combine after
# pooling, before the pin, tau only in the redundancy softmax; R23 a zero-norm key has cosine 0.
# --------------------------------------------------------------------------
def cosine_matrix(keys: np.ndarray) -> np.ndarray:
    """Cosine similarity of every pair of key rows (fp64), zero-norm rows -> 0 (R23)."""
    n = np.sqrt((keys * keys).sum(axis=1))
    safe = np.where(n > 0, n, 1.0)
    C = (keys @ keys.T) / safe[:, None] / safe[None, :]
    C[n == 0, :] = 0.0
    C[:, n == 0] = 0.0
    return C


def redundancy_raw_masked(keys: np.ndarray, mask: np.ndarray, p: float) -> np.ndarray:
    """The redundancy computation of PAPER.md:502 on the similarity entries allowed by `mask`
    ([T, T] bool): diagonal zeroed, per column the LAST (largest row index) entry > p zeroed,
    row sums, divided by the sequence length T. mask = all-True is the paper's original (naive)
    score; the block-diagonal mask is the lightning score."""
    T = keys.shape[0]
    C = np.where(mask, cosine_matrix(keys), 0.0)
    np.fill_diagonal(C, 0.0)
    for j in range(T):
        above = np.nonzero(C[:, j] > p)[0]
        if len(above):
            C[above[-1], j] = 0.0
    return C.sum(axis=1) / T


def lightning_redundancy_raw(keys: np.ndarray, b: int, p: float) -> np.ndarray:
    """Lightning redundancy, written per block of b tokens (the last block may
    be partial: only the T valid tokens take part, R20)."""
    T = keys.shape[0]
    r = np.zeros(T)
    for j0 in range(0, T, b):
        blk = keys[j0:min(T, j0 + b)]
        C = cosine_matrix(blk)
        np.fill_diagonal(C, 0.0)
        for j in range(C.shape[1]):
            above = np.nonzero(C[:, j] > p)[0]
            if len(above):
                C[above[-1], j] = 0.0
        r[j0:j0 + len(blk)] = C.sum(axis=1)
    return r / T


def softmax_temperature(x: np.ndarray, tau: float) -> np.ndarray:
    """softmax(x / tau) over the sequence, max-subtracted."""
    z = x / tau
    e = np.exp(z - z.max())
    return e / e.sum()


def combine_redundancy(s_pooled: np.ndarray, r_raw: np.ndarray, lam: float, tau: float) -> np.ndarray:
    """S = S - lambda * R with R = softmax(r_raw / tau)."""
    return s_pooled - lam * softmax_temperature(r_raw, tau)


def unit_keys(geo: Geometry, k_pool_f64, table, T: int, l: int, h: int) -> np.ndarray:
    """The unit's T key rows in logical order (gathered through the block table)."""
    t = np.arange(T)
    return k_pool_f64[l, np.asarray(table)[t // geo.b], t % geo.b, h]


# --------------------------------------------------------------------------
# NEXT-2: global score — Alg. 2, PAPER.md:412-456 (§C.3), relocation PAPER.md:595 (§C.6)
# Readings: R24 F is fp32 [L, N_total, b, h_kv]; R25 "not the last block of the
# sequence" = the logical blocks i < N_max - 1 (the targets of the previous compaction; at the
# paper's trigger N = N_max that is every block but the last); R26 the update uses S before pooling
# and F keeps the updated, unpooled score; R27 an uncompressed request only stores S.
# --------------------------------------------------------------------------
def global_score_update(s: np.ndarray, f_layer: np.ndarray, table, T: int, h: int, b: int, n_max: int,
                        compressed: bool, alpha: float, n_prefix: int = 0) -> np.ndarray:
    """Alg. 2 over the blocks of one unit, written out block by block. Mutates
    f_layer ([N_total, b, h_kv] fp32) and returns the (possibly overwritten) scores. R31: the F entries
    of the request's shared prefix blocks (logical i < n_prefix) are read as history
    but not written: the blocks belong to several requests."""
    s = s.copy()
    N = (T + b - 1) // b
    for i in range(N):
        lo, hi = i * b, min(T, (i + 1) * b)
        si = s[lo:hi].copy()                                  # line 1: s_i of the i-th block
        p = int(table[i])                                     # line 2: offset through the block table
        if compressed and i < n_max - 1:                      # lines 6-8 (R25)
            fi = f_layer[p, :hi - lo, h].astype(np.float64)
            si = np.maximum(alpha * fi, si)
        if i >= n_prefix:
            f_layer[p, :hi - lo, h] = si                      # lines 4 / 10 (fp32 store, R24; R31)
        if compressed:
            s[lo:hi] = si                                     # line 11
    return s


def compact_gather_f(f_layer, table, targets, kept: np.ndarray, h: int, b: int):
    """The global-score rows follow their K/V rows: new[rank] = old[kept[rank]]."""
    table = np.asarray(table)
    targets = np.asarray(targets)
    fs = f_layer[table[kept // b], kept % b, h].copy()
    rank = np.arange(len(kept))
    f_layer[targets[rank // b], rank % b, h] = fs


# --------------------------------------------------------------------------
# a4: per-head top-l with the index tie rule — PAPER.md:85, :591 (§C.6)
# --------------------------------------------------------------------------
def select(s_final: np.ndarray, ell: int) -> np.ndarray:
    """Keep the ell positions first under (score desc, position desc) (R7), ascending."""
    T = len(s_final)
    order = np.lexsort((np.arange(T), s_final))   # ascending by score, then position
    kept = order[T - ell:]
    return np.sort(kept).astype(np.int32)


def kept_to_tag(kept: np.ndarray, N: int, b: int) -> np.ndarray:
    """Top-k tag T in {0,1}^{N x b}."""
    tag = np.zeros(N * b, np.int8)
    tag[kept] = 1
    return tag.reshape(N, b)


# --------------------------------------------------------------------------
# a5: compaction — Alg. 4
# --------------------------------------------------------------------------
def compact_alg4(k_layer: np.ndarray, v_layer: np.ndarray, table, targets, tag: np.ndarray, h: int, b: int):
    """Formulation A: the two-pointer sweep of Alg. 4, literally (in place).

    Read pointer p_r walks the request's logical slots block by block through the
    table; write pointer p_w walks the target sequence (targets[0..N_max-2], R9/R10).
    k_layer/v_layer: [N_total, b, h_kv, d] raw element arrays of ONE layer.
    """
    N = tag.shape[0]
    pr = (0, 0)      # (logical block i, slot)   Alg.4 line 1
    pw = (0, 0)      # (target index, slot)
    ell, s, i = 0, 0, 0                                           # line 2
    while i < N:                                                  # line 3
        if tag[i][ell % b] == 1:                                  # line 4
            kvec = k_layer[table[pr[0]], pr[1], h, :].copy()      # line 5
            vvec = v_layer[table[pr[0]], pr[1], h, :].copy()      # line 6
            k_layer[targets[pw[0]], pw[1], h, :] = kvec           # line 7
            v_layer[targets[pw[0]], pw[1], h, :] = vvec           # line 8
            s += 1                                                # line 9
            pw = (pw[0] + 1, 0) if s % b == 0 else (pw[0], pw[1] + 1)   # lines 10-14
        ell += 1                                                  # line 16
        if ell % b == 0:                                          # line 17
            pr = (pr[0] + 1, 0)
            i += 1
        else:
            pr = (pr[0], pr[1] + 1)


def compact_gather(k_layer, v_layer, table, targets, kept: np.ndarray, h: int, b: int):
    """Formulation B: snapshot the kept rows first, then write new[rank] = old[kept[rank]]."""
    table = np.asarray(table)
    targets = np.asarray(targets)
    src_blk, src_slot = table[kept // b], kept % b
    ks = k_layer[src_blk, src_slot, h, :].copy()
    vs = v_layer[src_blk, src_slot, h, :].copy()
    rank = np.arange(len(kept))
    k_layer[targets[rank // b], rank % b, h, :] = ks
    v_layer[targets[rank // b], rank % b, h, :] = vs


# --------------------------------------------------------------------------
# a6: tables, ref counts, freed list — PAPER.md:64 (§4.1), :138 (§4.5); Fig. 1 caption :22
# --------------------------------------------------------------------------
@dataclass
class FinalizeOut:
    tables: np.ndarray
    new_num_blocks: np.ndarray
    freed: np.ndarray
    free_stack: np.ndarray
    free_top: int
    ref_counts: np.ndarray | None


def finalize(geo: Geometry, prm: Params, pl: Plan, tables, ref_counts, free_stack, free_top) -> FinalizeOut:
    """New table = targets ++ [reserved] (N_max entries; the N_max-th block is reserved
    for decoding). Freed = each request's private blocks that are neither
    targets nor reserved, ascending logical index, requests in input order; then the
    shared blocks whose count this call drove to 0, ascending id. Shared blocks get
    ref -= 1. With ref counts: fresh targets/reserved -> 1, freed private -> 0.
    The freed list is pushed onto the free stack in list order."""
    R = len(pl.n_blocks)
    nm1 = prm.n_max - 1
    tables = tables.copy()
    refs = None if ref_counts is None else ref_counts.copy()
    stack = free_stack.copy()
    top = int(free_top) - sum(len(f) for f in pl.fresh)
    freed = []
    zeroed = set()
    for r in range(R):
        N, n_prefix = int(pl.n_blocks[r]), int(pl.n_prefix[r])
        old = [int(x) for x in tables[r, :N]]
        first_priv_free = max(n_prefix, nm1) + 1
        for j in range(first_priv_free, N):
            freed.append(old[j])
            if refs is not None:
                refs[old[j]] = 0
        if refs is not None:
            for j in range(n_prefix):
                refs[old[j]] -= 1
                if refs[old[j]] == 0:
                    zeroed.add(old[j])
            for bid in pl.fresh[r]:
                refs[bid] = 1
        tables[r, :nm1] = pl.targets[r]
        tables[r, nm1] = pl.reserved[r]
    freed.extend(sorted(zeroed))
    for bid in freed:
        stack[top] = bid
        top += 1
    return FinalizeOut(tables=tables, new_num_blocks=np.full(R, prm.n_max, np.int32),
                       freed=np.asarray(freed, np.int32), free_stack=stack, free_top=top,
                       ref_counts=refs)


# --------------------------------------------------------------------------
# the whole step
# --------------------------------------------------------------------------
@dataclass
class CompressOut:
    status: int
    k_cache: np.ndarray = None
    v_cache: np.ndarray = None
    new_lens: np.ndarray = None      # [R, L, h_kv]
    kept: dict = None                # (r, l, h) -> ascending kept positions
    scores: dict = None              # (r, l, h) -> raw s (pre-pool) fp64
    fin: FinalizeOut = None
    redundancy: dict = None          # (r, l, h) -> lightning r_raw (pre-softmax) fp64 (F_REDUNDANCY)
    f_cache: np.ndarray = None       # F after the step (F_GLOBAL_SCORE)
    global_scores: dict = None       # (r, l, h) -> S after Alg. 2 (pre-pool) (F_GLOBAL_SCORE)
    plan: Plan = None


def compress(geo: Geometry, prm: Params, k_cache, v_cache, q_cache, q_slots, seq_lens, tables, budgets,
             ref_counts=None, free_stack=None, free_top=0, kept_override=None, blockwise=False,
             free_capacity=None, freed_capacity=None, units=None, f_cache=None, is_compressed=None,
             window_lse_in=None) -> CompressOut:
    """Steps 1-9 of SURVEY.md §8(c) for every request r (input order), layer l, KV head h.

    kept_override: optional dict (r, l, h) -> kept list, used to drive compaction with
    a kept set chosen elsewhere (the 'bytes' parity rule). units: optional subset of
    (r, l, h) to score (for sampled checks); compaction then needs kept_override.
    window_lse_in: optional [L][M][w][h_q] natural-log normalisers (NEXT-4, ZPC_F_LSE_INPUT).
    """
    pl = plan(geo, prm, seq_lens, tables, budgets, ref_counts, free_stack, free_top, q_slots,
              free_capacity, freed_capacity)
    if pl.status != OK:
        return CompressOut(status=pl.status, plan=pl)
    R = len(seq_lens)
    if prm.flags & F_VALIDATE:
        # R33: every K row t < T of every unit and every window query row must be finite (the selection
        # order of PAPER.md:591 is undefined for NaN scores); a batch-level check after plan's
        kf_all, qf_all = widen(k_cache, geo.dtype), widen(q_cache, geo.dtype)
        G = geo.h_q // geo.h_kv
        for r in range(R):
            T, tb = int(seq_lens[r]), np.asarray(tables[r])
            t = np.arange(T)
            for l in range(geo.L):
                for h in range(geo.h_kv):
                    rows = kf_all[l, tb[t // geo.b], t % geo.b, h]
                    qw = qf_all[l, int(q_slots[r]), :, h * G:(h + 1) * G]
                    if not (np.isfinite(rows).all() and np.isfinite(qw).all()):
                        return CompressOut(status=ERR_NONFINITE, plan=pl)
    k_out = k_cache.copy()
    v_out = v_cache.copy()
    use_global = bool(prm.flags & F_GLOBAL_SCORE)
    f_out = f_cache.copy() if use_global else None
    qf = widen(q_cache, geo.dtype)
    kf = widen(k_cache, geo.dtype)
    new_lens = np.zeros((R, geo.L, geo.h_kv), np.int32)
    kept_all, scores, redund, gscores = {}, {}, {}, {}
    for r in range(R):
        T = int(seq_lens[r])
        for l in range(geo.L):
            for h in range(geo.h_kv):
                ell = min(T, int(budgets[r, l, h]))
                new_lens[r, l, h] = ell
                key = (r, l, h)
                if kept_override is not None and key in kept_override:
                    kept = np.asarray(kept_override[key], np.int32)
                    if use_global:   # F is still updated by Alg. 2 before it is relocated
                        s = unit_scores(geo, qf, kf, tables[r], T, int(q_slots[r]), l, h, blockwise, window_lse_in)
                        gscores[key] = global_score_update(s, f_out[l], tables[r], T, h, geo.b, prm.n_max,
                                                           bool(is_compressed[r]), prm.alpha,
                                                           int(pl.n_prefix[r]))
                else:
                    if units is not None and key not in units:
                        continue
                    s = unit_scores(geo, qf, kf, tables[r], T, int(q_slots[r]), l, h, blockwise, window_lse_in)
                    scores[key] = s
                    if use_global:
                        s = global_score_update(s, f_out[l], tables[r], T, h, geo.b, prm.n_max,
                                                bool(is_compressed[r]), prm.alpha, int(pl.n_prefix[r]))
                        gscores[key] = s
                    # R32: with F_POOL_FIRST only a request's first compression pools
                    first = not (prm.flags & F_POOL_FIRST) or not bool(is_compressed[r])
                    sp = max_pool(s, prm.pool_kernel if first else 1)
                    if prm.flags & F_REDUNDANCY:
                        rr = lightning_redundancy_raw(unit_keys(geo, kf, tables[r], T, l, h), geo.b, prm.sim_p)
                        redund[key] = rr
                        sp = combine_redundancy(sp, rr, prm.lam, prm.tau)
                    kept = select(pin_window(sp, T, geo.w), ell)
                kept_all[key] = kept
    for r in range(R):
        N = int(pl.n_blocks[r])
        for l in range(geo.L):
            for h in range(geo.h_kv):
                key = (r, l, h)
                if key not in kept_all:
                    continue
                compact_gather(k_out[l], v_out[l], tables[r], pl.targets[r], kept_all[key], h, geo.b)
                if use_global:
                    compact_gather_f(f_out[l], tables[r], pl.targets[r], kept_all[key], h, geo.b)
    fin = finalize(geo, prm, pl, tables, ref_counts, free_stack, free_top)
    return CompressOut(status=OK, k_cache=k_out, v_cache=v_out, new_lens=new_lens, kept=kept_all,
                       scores=scores, fin=fin, plan=pl, redundancy=redund, f_cache=f_out, global_scores=gscores)
