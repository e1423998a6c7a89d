// a0 plan and a6 finalize: integer block bookkeeping of the compression step.
//   plan:     trigger check (§4.1), prefix-aware targets (§4.5),
//             fresh pops assigned by an exclusive scan in request order (deterministic).
//   finalize: new tables = targets ++ [reserved]; freed list (private blocks ascending logical
//             index per request, then shared blocks driven to ref 0 ascending id); ref counts
//             (PAPER.md:138); push onto the free stack. No atomics decide any order.
#include "internal.h"

namespace zpc {

namespace {

constexpr int kScanThreads = 1024;

// Block-wide exclusive scan of one int per thread; returns the exclusive prefix and the total.
template <int NT>
__device__ int block_exclusive_scan(int v, int* total, int* smem /*[NT/32 + 1]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = (lane < NT / 32) ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) smem[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  int warp_off = warp ? smem[warp - 1] : 0;
  int tot = smem[NT / 32 - 1];
  __syncthreads();
  *total = tot;
  return warp_off + x - v;
}

__device__ __forceinline__ int block_or(int v, int* sh) {
  v = __syncthreads_or(v);
  (void)sh;
  return v;
}

// Request r (the whole CTA): validation in the documented order + per-request counts.
__device__ void plan_req_body(const Call& c, const int r) {
  __shared__ int s_first_private;
  __shared__ int s_err;
  const int nm1 = c.n_max - 1;
  const int T = c.seq_lens[r];
  int err = ZPC_OK;
  int N = 0, np = 0;
  const int* table = c.tables + (size_t)r * c.table_stride;
  const int slot = c.q_slots[r];
  if (slot < 0 || slot >= c.M) err = ZPC_ERR_BAD_SLOT;
  else if (T > c.max_seq_len) err = ZPC_ERR_SEQ_TOO_LONG;
  else {
    N = (T + c.b - 1) / c.b;
    if (N > c.table_stride) err = ZPC_ERR_BAD_TABLE;
    else if (N < c.n_max) err = ZPC_ERR_NOT_TRIGGERED;
  }
  if (err == ZPC_OK) {
    int bad = 0;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      int id = table[j];
      bad |= (id < 0 || id >= c.N_total);
    }
    if (__syncthreads_or(bad)) err = ZPC_ERR_BAD_TABLE;
  }
  if (err == ZPC_OK && (c.flags & ZPC_F_VALIDATE)) {
    int dup = 0;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      int id = table[j];
      for (int k = j + 1; k < N; ++k) dup |= (table[k] == id);
    }
    if (__syncthreads_or(dup)) err = ZPC_ERR_BAD_TABLE;
  }
  if (err == ZPC_OK && (c.flags & ZPC_F_PREFIX)) {
    if (threadIdx.x == 0) s_first_private = N;
    __syncthreads();
    for (int j = threadIdx.x; j < N; j += blockDim.x)
      if (c.ref_counts[table[j]] <= 1) atomicMin(&s_first_private, j);
    __syncthreads();
    np = s_first_private;
    int bad = 0;
    for (int j = np + threadIdx.x; j < N; j += blockDim.x) bad |= (c.ref_counts[table[j]] > 1);
    if (__syncthreads_or(bad)) err = ZPC_ERR_BAD_TABLE;
  }
  if (err == ZPC_OK) {
    const int kmax = nm1 * c.b;
    const int* bud = c.budgets + (size_t)r * c.L * c.h_kv;
    int bad = 0;
    for (int i = threadIdx.x; i < c.L * c.h_kv; i += blockDim.x) bad |= (bud[i] < c.w || bud[i] > kmax);
    if (__syncthreads_or(bad)) err = ZPC_ERR_BAD_BUDGET;
  }
  (void)s_err;
  // occurrences of each shared block in this batch (exact capacity check, R18)
  if (err == ZPC_OK)
    for (int j = threadIdx.x; j < np; j += blockDim.x) atomicAdd(&c.ws.marks[table[j]], 1);
  if (threadIdx.x == 0) {
    c.ws.req_err[r] = err;
    c.ws.n_blocks[r] = N;
    c.ws.n_prefix[r] = np;
  }
}
// One CTA per request.
__global__ void __launch_bounds__(256) k_plan_req(Call c) { plan_req_body(c, blockIdx.x); }

// Single CTA: first failing request -> status; scans; batch checks; target assignment.
__device__ void plan_scan_body(const Call& c) {
  __shared__ int sm[kScanThreads / 32 + 1];
  __shared__ int s_minr;
  const int nm1 = c.n_max - 1;
  if (threadIdx.x == 0) s_minr = 0x7fffffff;
  __syncthreads();
  for (int r = threadIdx.x; r < c.R; r += blockDim.x)
    if (c.ws.req_err[r] != ZPC_OK) atomicMin(&s_minr, r);
  __syncthreads();
  if (s_minr != 0x7fffffff) {
    if (threadIdx.x == 0) *c.status = c.ws.req_err[s_minr];
    return;
  }
  // exclusive scans over requests (chunks of kScanThreads)
  int fresh_base = 0, priv_base = 0, zeroed = 0;
  if (c.ref_counts && (c.flags & ZPC_F_PREFIX)) {
    int z = 0;
    for (int i = threadIdx.x; i < c.N_total; i += blockDim.x) {
      const int occ = c.ws.marks[i];
      z += (occ > 0 && occ == c.ref_counts[i]);
    }
    block_exclusive_scan<kScanThreads>(z, &zeroed, sm);
  }
  for (int r0 = 0; r0 < c.R; r0 += kScanThreads) {
    const int r = r0 + threadIdx.x;
    int nf = 0, npv = 0;
    if (r < c.R) {
      const int N = c.ws.n_blocks[r], np = c.ws.n_prefix[r];
      const int res_idx = max(np, nm1);
      nf = min(np, nm1) + (res_idx >= N ? 1 : 0);
      npv = max(0, N - 1 - res_idx);
    }
    int tf, tp;
    int of = block_exclusive_scan<kScanThreads>(nf, &tf, sm);
    int op = block_exclusive_scan<kScanThreads>(npv, &tp, sm);
    if (r < c.R) {
      c.ws.fresh_off[r] = fresh_base + of;
      c.ws.priv_off[r] = priv_base + op;
    }
    fresh_base += tf;
    priv_base += tp;
  }
  const int top = *c.free_top;
  int st = ZPC_OK;
  if (fresh_base > top) st = ZPC_ERR_NO_FREE_BLOCKS;
  else if ((long long)priv_base + zeroed > c.freed_capacity) st = ZPC_ERR_CAPACITY;
  else if ((long long)top - fresh_base + priv_base + zeroed > c.free_capacity) st = ZPC_ERR_CAPACITY;
  if (st != ZPC_OK) {
    if (threadIdx.x == 0) *c.status = st;
    return;
  }
  // targets[r][j]: fresh pops from the stack top in (request, target index) order, reserved last
  const long long total = (long long)c.R * c.n_max;
  for (long long i = threadIdx.x; i < total; i += blockDim.x) {
    const int r = (int)(i / c.n_max), j = (int)(i % c.n_max);
    const int N = c.ws.n_blocks[r], np = c.ws.n_prefix[r];
    const int* table = c.tables + (size_t)r * c.table_stride;
    const int off = c.ws.fresh_off[r];
    if (j < nm1) {
      c.ws.targets[(size_t)r * nm1 + j] = (j < np) ? c.free_stack[top - 1 - (off + j)] : table[j];
    } else {
      const int res_idx = max(np, nm1);
      c.ws.reserved[r] = (res_idx < N) ? table[res_idx] : c.free_stack[top - 1 - (off + min(np, nm1))];
    }
  }
  if (threadIdx.x == 0) {
    c.ws.glob[0] = fresh_base;
    c.ws.glob[1] = priv_base;
    c.ws.glob[2] = top - fresh_base;
    *c.status = ZPC_OK;
  }
}
__global__ void __launch_bounds__(kScanThreads) k_plan_scan(Call c) { plan_scan_body(c); }
// Single-request calls (R <= kSmallR): both steps in one CTA -- one launch instead of two. paper_op step (graph)
// with plan and finalize fused at R <= 4: 1 request 0.1873 -> 0.1851 ms, 4 requests 0.6127 -> 0.6158 (the
// requests in turn cost more than the launch saved), hence R = 1 only
constexpr int kSmallR = 1;
__global__ void __launch_bounds__(kScanThreads) k_plan_small(Call c) {
  for (int r = 0; r < c.R; ++r) {
    plan_req_body(c, r);
    __syncthreads();   // its shared scratch is reused by the next request; its global outputs feed the scan
  }
  plan_scan_body(c);
}

// Request r (the whole CTA): freed private list, ref counts, then the new table.
__device__ void finalize_req_body(const Call& c, const int r) {
  const int nm1 = c.n_max - 1;
  const int N = c.ws.n_blocks[r], np = c.ws.n_prefix[r];
  int* table = c.tables + (size_t)r * c.table_stride;
  const int first = max(np, nm1) + 1;
  const int poff = c.ws.priv_off[r];
  // phase 1: everything that reads the old table
  for (int j = first + threadIdx.x; j < N; j += blockDim.x) {
    const int id = table[j];
    c.freed[poff + (j - first)] = id;
    if (c.ref_counts) c.ref_counts[id] = 0;
  }
  if (c.ref_counts && (c.flags & ZPC_F_PREFIX)) {
    for (int j = threadIdx.x; j < np; j += blockDim.x) {
      const int id = table[j];
      atomicSub(&c.ref_counts[id], 1);
    }
  }
  __syncthreads();
  // phase 2: new table (first N_max entries) and fresh-block refs
  const int* tg = c.ws.targets + (size_t)r * nm1;
  for (int j = threadIdx.x; j < nm1; j += blockDim.x) {
    table[j] = tg[j];
    if (c.ref_counts && j < np) c.ref_counts[tg[j]] = 1;
  }
  if (threadIdx.x == 0) {
    table[nm1] = c.ws.reserved[r];
    if (c.ref_counts && max(np, nm1) >= N) c.ref_counts[c.ws.reserved[r]] = 1;
    c.new_num_blocks[r] = c.n_max;
  }
}
// One CTA per request.
__global__ void __launch_bounds__(256) k_finalize_req(Call c) {
  if (*c.status != ZPC_OK) return;
  finalize_req_body(c, blockIdx.x);
}

// Single CTA: shared blocks driven to zero (ascending id), num_freed, free-stack push.
__device__ void finalize_tail_body(const Call& c) {
  __shared__ int sm[kScanThreads / 32 + 1];
  const int priv = c.ws.glob[1];
  int base = priv;
  if (c.ref_counts && (c.flags & ZPC_F_PREFIX)) {
    for (int i0 = 0; i0 < c.N_total; i0 += kScanThreads) {
      const int i = i0 + threadIdx.x;
      const int m = (i < c.N_total) ? (c.ws.marks[i] > 0 && c.ref_counts[i] == 0) : 0;
      int tot;
      const int off = block_exclusive_scan<kScanThreads>(m, &tot, sm);
      if (m) c.freed[base + off] = i;
      base += tot;
    }
  }
  const int nfreed = base;
  __syncthreads();
  __threadfence_block();
  const int top_base = c.ws.glob[2];
  for (int i = threadIdx.x; i < nfreed; i += blockDim.x) c.free_stack[top_base + i] = c.freed[i];
  if (threadIdx.x == 0) {
    *c.num_freed = nfreed;
    *c.free_top = top_base + nfreed;
    c.ws.glob[3] = nfreed - priv;
  }
}
__global__ void __launch_bounds__(kScanThreads) k_finalize_tail(Call c) {
  if (*c.status != ZPC_OK) return;
  finalize_tail_body(c);
}
__global__ void __launch_bounds__(kScanThreads) k_finalize_small(Call c) {
  if (*c.status != ZPC_OK) return;
  for (int r = 0; r < c.R; ++r) finalize_req_body(c, r);
  __syncthreads();
  __threadfence_block();   // every request's ref-count updates before the zeroed-block scan reads them
  finalize_tail_body(c);
}

}  // namespace

// ZPC_F_VALIDATE: every Q and K element the call reads must be finite (PAPER.md:591 pins the window at
// +inf and the selection orders finite scores; a NaN key or query would make that order undefined).
// One CTA per (unit, 2048-token slab): the unit's K rows t < T through the block table and, in slab 0, its
// G*w window query rows; 16-B vectors, exponent-all-ones test (bf16 0x7F80, fp32 0x7F800000). Runs after
// plan; a failure sets *status = ZPC_ERR_NONFINITE only if plan left it OK (batch-level check after the
// per-request ones), so every later stage returns at entry and nothing is mutated.
constexpr int kValSlab = 2048;
__global__ void __launch_bounds__(256) k_validate(Call c) {
  if (*c.status != ZPC_OK) return;
  const int unit = blockIdx.x;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int t0 = blockIdx.y * kValSlab;
  if (t0 >= T) return;
  const int esz = c.dtype == ZPC_BF16 ? 2 : 4;
  const int vpr = c.d * esz / 16;                       // 16-B vectors per row
  const uint4* K = reinterpret_cast<const uint4*>(c.k_cache);
  const int32_t* table = c.tables + (size_t)r * c.table_stride;
  auto bad = [&](uint4 v) -> bool {
    if (esz == 2) {
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      bool b = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) b |= ((w[i] & 0x7F80u) == 0x7F80u) | ((w[i] & 0x7F800000u) == 0x7F800000u);
      return b;
    }
    return ((v.x & 0x7F800000u) == 0x7F800000u) | ((v.y & 0x7F800000u) == 0x7F800000u) |
           ((v.z & 0x7F800000u) == 0x7F800000u) | ((v.w & 0x7F800000u) == 0x7F800000u);
  };
  bool found = false;
  const int n = (min(T, t0 + kValSlab) - t0) * vpr;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int t = t0 + i / vpr, e = i % vpr;
    found |= bad(K[kv_row(c, l, table[t / c.b], t % c.b, h) * esz / 16 + e]);
  }
  if (blockIdx.y == 0) {
    const uint4* Q = reinterpret_cast<const uint4*>(c.q_cache);
    const int slot = c.q_slots[r];
    const int nq = c.w * c.G * vpr;
    for (int i = threadIdx.x; i < nq; i += blockDim.x) {
      const int row = i / vpr, e = i % vpr, u = row / c.G, g = row % c.G;
      found |= bad(Q[q_row(c, l, slot, u, h * c.G + g) * esz / 16 + e]);
    }
  }
  if (__syncthreads_or(found) && threadIdx.x == 0) atomicCAS(c.status, ZPC_OK, ZPC_ERR_NONFINITE);
}

cudaError_t launch_plan(const Call& c, cudaStream_t s) {
  if (c.ref_counts && (c.flags & ZPC_F_PREFIX))
    cudaMemsetAsync(c.ws.marks, 0, sizeof(int32_t) * (size_t)c.N_total, s);
  if (c.R <= kSmallR) {
    k_plan_small<<<1, kScanThreads, 0, s>>>(c);
  } else {
    k_plan_req<<<c.R, 256, 0, s>>>(c);
    k_plan_scan<<<1, kScanThreads, 0, s>>>(c);
  }
  if ((c.flags & ZPC_F_VALIDATE) && c.R > 0) {
    const dim3 grid((unsigned)(c.R * c.L * c.h_kv), (unsigned)((c.max_seq_len + kValSlab - 1) / kValSlab));
    k_validate<<<grid, 256, 0, s>>>(c);
  }
  return cudaGetLastError();
}

cudaError_t launch_finalize(const Call& c, cudaStream_t s) {
  if (c.R <= kSmallR) {
    k_finalize_small<<<1, kScanThreads, 0, s>>>(c);
  } else {
    k_finalize_req<<<c.R, 256, 0, s>>>(c);
    k_finalize_tail<<<1, kScanThreads, 0, s>>>(c);
  }
  return cudaGetLastError();
}

}  // namespace zpc
