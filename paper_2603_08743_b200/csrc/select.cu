// a3 + a4: MaxPool1D + window pin + per-head top-l with the
// index tie rule (R7: score desc, position desc), emitted ascending. One CTA per unit (r, l, h).
// Selection is an exact 4-pass MSB radix select over order-preserving uint32 keys held in shared
// memory, followed by a deterministic two-scan emission — no sort, no atomics decide the result.
#include <cstdlib>

#include "internal.h"

namespace zpc {
namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

// fp32 -> uint32 with the same order (for finite values and +inf); -0 canonicalised to +0.
__device__ __forceinline__ uint32_t orderable(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ int warp_incl_scan(int x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// exclusive prefix over threads in index order; *total = sum
__device__ int block_excl(int v, int* sm, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = warp_incl_scan(v);
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = sm[lane];
    s = warp_incl_scan(s);
    sm[lane] = s;
  }
  __syncthreads();
  const int off = (warp ? sm[warp - 1] : 0) + x - v;
  *total = sm[kWarps - 1];
  __syncthreads();
  return off;
}

__device__ float block_max(float v, float* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  float x = lane < kWarps ? sm[lane] : -INFINITY;
#pragma unroll
  for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  __syncthreads();
  return x;
}
__device__ float block_sum(float v, float* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  float x = lane < kWarps ? sm[lane] : 0.f;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  return x;
}

// GK = false: the unit's keys live in shared memory (T <= kSelectSmemMaxT); GK = true (longer units, up to
// ZPC_MAX_SEQ_LEN): in the workspace region select_keys [units][max_seq_len] (L2-resident while the CTA works
// on it); every step is the same code on the other array.
template <bool GK>
__global__ void __launch_bounds__(kThreads) k_select(Call c) {
  if (*c.status != ZPC_OK) return;
  extern __shared__ uint32_t keys_smem[];       // [T] (GK = false)
  __shared__ int hist[256];
  __shared__ int sm[kWarps];
  __shared__ float fsm[kWarps];
  __shared__ uint32_t s_prefix;
  __shared__ int s_need;

  const int unit = blockIdx.x;
  uint32_t* keys = GK ? c.ws.select_keys + (size_t)unit * c.max_seq_len : keys_smem;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int ell = min(T, c.budgets[unit]);
  if (threadIdx.x == 0) c.new_lens[unit] = ell;
  const float* S = c.ws.scores + (size_t)unit * c.max_seq_len;
  // R32: ZPC_F_POOL_FIRST pools only a request's first compression
  const int half = ((c.flags & ZPC_F_POOL_FIRST) && c.is_compressed[r]) ? 0 : c.pool_kernel / 2;

  // NEXT-2 (ZPC_F_GLOBAL_SCORE): Alg. 2 over the unit's blocks before pooling
  // (PAPER.md:487): F <- S for a request never compressed; otherwise S <- max(alpha F, S) on the
  // logical blocks < N_max-1 (the previous targets, R25), F <- S, and S is overwritten (line 11)
  if (c.flags & ZPC_F_GLOBAL_SCORE) {
    const bool comp = c.is_compressed[r] != 0;
    const int32_t* table = c.tables + (size_t)r * c.table_stride;
    float* Sw = c.ws.scores + (size_t)unit * c.max_seq_len;
    const size_t fplane = (size_t)l * c.N_total * c.b * c.h_kv + h;
    // R31: F of the shared prefix blocks (logical < n_prefix) is history only, never stored (several
    // requests of the batch own the block; their updates would race)
    const int npre = (c.flags & ZPC_F_PREFIX) ? c.ws.n_prefix[r] : 0;
    for (int t = threadIdx.x; t < T; t += kThreads) {
      const int i = t / c.b;
      float* fp = c.f_cache + fplane + ((size_t)table[i] * c.b + (t - i * c.b)) * c.h_kv;
      float v = Sw[t];
      if (comp && i < c.n_max - 1) v = fmaxf(c.global_alpha * *fp, v);
      if (i >= npre) *fp = v;
      if (comp) Sw[t] = v;
    }
    __syncthreads();
  }
  // NEXT-1 (ZPC_F_REDUNDANCY): R = softmax(r / tau) over the sequence; the pooled
  // score becomes S - lambda * R before the pin (R22)
  const bool red = (c.flags & ZPC_F_REDUNDANCY) != 0;
  const float* rr = c.ws.redund + (size_t)unit * c.max_seq_len;
  float rmax = 0.f, rscale = 0.f;
  const float inv_tau = red ? 1.0f / c.red_tau : 0.f;
  if (red) {
    float m = -INFINITY;
    for (int t = threadIdx.x; t < T; t += kThreads) m = fmaxf(m, rr[t]);
    rmax = block_max(m, fsm);
    float z = 0.f;
    for (int t = threadIdx.x; t < T; t += kThreads) z += expf((rr[t] - rmax) * inv_tau);
    rscale = c.red_lambda / block_sum(z, fsm);      // lambda / sum
  }
  // load + pool (+ redundancy) + pin -> keys
  for (int t = threadIdx.x; t < T; t += kThreads) {
    float v;
    if (t >= T - c.w) {
      v = __int_as_float(0x7f800000);            // +inf: observation window is always kept
    } else {
      v = S[t];
      const int lo = max(0, t - half), hi = min(T - 1, t + half);
      for (int j = lo; j <= hi; ++j) v = fmaxf(v, S[j]);
      if (red) v -= rscale * expf((rr[t] - rmax) * inv_tau);
    }
    keys[t] = orderable(v);
  }
  if (threadIdx.x == 0) { s_prefix = 0; s_need = ell; }
  __syncthreads();

  // MSB radix select of the ell-th largest key
  uint32_t mask = 0;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += kThreads) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
    for (int t = threadIdx.x; t < T; t += kThreads) {
      const uint32_t k = keys[t];
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // find digit d: count(>d) < need <= count(>=d), scanning from 255 down (warp 0)
      const int lane = threadIdx.x;
      // each lane owns 8 consecutive digits, lane 0 the highest
      int cnt[8];
      int sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { cnt[i] = hist[255 - (lane * 8 + i)]; sum += cnt[i]; }
      int incl = warp_incl_scan(sum);
      const int excl = incl - sum;                 // count of keys with digit above this lane's range
      const int need = s_need;
      int found = -1, above = 0;
      int run = excl;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (found < 0 && run < need && run + cnt[i] >= need) { found = 255 - (lane * 8 + i); above = run; }
        run += cnt[i];
      }
      const unsigned ball = __ballot_sync(0xffffffffu, found >= 0);
      const int src = __ffs(ball) - 1;
      const int d = __shfl_sync(0xffffffffu, found, src);
      const int ab = __shfl_sync(0xffffffffu, above, src);
      if (lane == 0) { s_prefix = prefix | ((uint32_t)d << shift); s_need = need - ab; }
    }
    mask |= 0xffu << shift;
    __syncthreads();
  }
  const uint32_t kstar = s_prefix;
  const int need_eq = s_need;   // how many keys == kstar to keep: the latest positions

  // emission: contiguous chunk per thread
  const int chunk = (T + kThreads - 1) / kThreads;
  const int t0 = min(T, threadIdx.x * chunk), t1 = min(T, t0 + chunk);
  int eq = 0;
  for (int t = t0; t < t1; ++t) eq += (keys[t] == kstar);
  int eq_tot;
  const int eq_before = block_excl(eq, sm, &eq_tot);
  int eq_after = eq_tot - eq_before - eq;      // equal keys at later positions than this chunk
  int kept_here = 0;
  for (int t = t1 - 1; t >= t0; --t) {
    const uint32_t k = keys[t];
    bool keep = k > kstar;
    if (k == kstar) { keep = eq_after < need_eq; ++eq_after; }
    kept_here += keep;
    keys[t] = keep ? 1u : 0u;                  // reuse as flag (own chunk only)
  }
  int kept_tot;
  const int out0 = block_excl(kept_here, sm, &kept_tot);
  int32_t* out = c.ws.kept + (size_t)unit * c.ws.kept_stride;
  int o = out0;
  for (int t = t0; t < t1; ++t)
    if (keys[t]) { ZPC_CHECK(o < ell && t < T); out[o++] = t; }
}


// Register-resident variant for T <= kThreads * CH (the configs: CH = 8 / 16 / 32 for T = 8K / 16K / 32K).
// Same result as k_select, bit for bit (same keys, same radix digits, same tie rule and emission); the
// differences are where the keys live and how the histogram is built:
//  * S is staged once through shared memory (coalesced loads, bank-padded index t + t/32), each thread
//    pools its contiguous chunk of CH positions from there and keeps the orderable keys in registers;
//  * a warp whose participating keys share one digit adds its count with a single shared atomic -- the
//    first digits (sign + top exponent bits) are shared by nearly every score, so per-element atomics
//    serialised on one or two bins; other warps add per element. Measured on the 7B batch: 0.81 ms
//    (k_select) -> 0.69 (__match_any_sync grouping) -> 0.62 (this vote); vote + match fallback 0.82.

// block-wide helpers for an NT-thread CTA (NT a multiple of 32, <= 1024)
template <int NT>
__device__ int block_excl_t(int v, int* sm, int* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = warp_incl_scan(v);
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = lane < NW ? sm[lane] : 0;
    s = warp_incl_scan(s);
    if (lane < NW) sm[lane] = s;
  }
  __syncthreads();
  const int off = (warp ? sm[warp - 1] : 0) + x - v;
  *total = sm[NW - 1];
  __syncthreads();
  return off;
}
template <int NT>
__device__ float block_max_t(float v, float* sm) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  float x = lane < NW ? sm[lane] : -INFINITY;
#pragma unroll
  for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  __syncthreads();
  return x;
}
template <int NT>
__device__ float block_sum_t(float v, float* sm) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  float x = lane < NW ? sm[lane] : 0.f;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  return x;
}

__device__ __forceinline__ int pidx(int t) { return t + (t >> 5); }

template <int NT, int CH>
__device__ __forceinline__ void select_reg_unit(const Call& c, const int unit) {
  extern __shared__ float sS[];                 // [pidx(T)] staged S (padded)
  __shared__ int hist[256];
  __shared__ int sm[NT / 32];
  __shared__ float fsm[NT / 32];
  __shared__ uint32_t s_prefix;
  __shared__ int s_need;

  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int ell = min(T, c.budgets[unit]);
  if (threadIdx.x == 0) c.new_lens[unit] = ell;
  // R32: ZPC_F_POOL_FIRST pools only a request's first compression
  const int half = ((c.flags & ZPC_F_POOL_FIRST) && c.is_compressed[r]) ? 0 : c.pool_kernel / 2;

  // NEXT-2 (ZPC_F_GLOBAL_SCORE): Alg. 2 as in k_select (R25-R27), S updated in place
  float* Sw = c.ws.scores + (size_t)unit * c.max_seq_len;
  if (c.flags & ZPC_F_GLOBAL_SCORE) {
    const bool comp = c.is_compressed[r] != 0;
    const int32_t* table = c.tables + (size_t)r * c.table_stride;
    const size_t fplane = (size_t)l * c.N_total * c.b * c.h_kv + h;
    const int npre = (c.flags & ZPC_F_PREFIX) ? c.ws.n_prefix[r] : 0;   // R31: shared blocks' F read only
    for (int t = threadIdx.x; t < T; t += NT) {
      const int i = t / c.b;
      float* fp = c.f_cache + fplane + ((size_t)table[i] * c.b + (t - i * c.b)) * c.h_kv;
      float v = Sw[t];
      if (comp && i < c.n_max - 1) v = fmaxf(c.global_alpha * *fp, v);
      if (i >= npre) *fp = v;
      if (comp) Sw[t] = v;
    }
    __syncthreads();
  }
  // NEXT-1 (ZPC_F_REDUNDANCY): lambda * softmax(r / tau) subtracted after pooling
  const bool red = (c.flags & ZPC_F_REDUNDANCY) != 0;
  const float* rr = c.ws.redund + (size_t)unit * c.max_seq_len;
  float rmax = 0.f, rscale = 0.f;
  const float inv_tau = red ? 1.0f / c.red_tau : 0.f;
  if (red) {
    float m = -INFINITY;
    for (int t = threadIdx.x; t < T; t += NT) m = fmaxf(m, rr[t]);
    rmax = block_max_t<NT>(m, fsm);
    float z = 0.f;
    for (int t = threadIdx.x; t < T; t += NT) z += expf((rr[t] - rmax) * inv_tau);
    rscale = c.red_lambda / block_sum_t<NT>(z, fsm);
  }
  for (int t = threadIdx.x; t < T; t += NT) sS[pidx(t)] = Sw[t];
  if (threadIdx.x == 0) { s_prefix = 0; s_need = ell; }
  __syncthreads();

  // pool (+ redundancy) + pin of this thread's chunk [t0, t0 + CH) -> keys in registers
  const int t0 = threadIdx.x * CH;
  uint32_t key[CH];
  if (half == 3) {
    // k_p = 7 (the configs' pool): the chunk and its 3 neighbours on each side are loaded once
    // (out-of-range = -inf, PAPER.md:482 reading R6), then max over e[i..i+6] by a 2-4-7 doubling tree
    // (max is exact, so the result is bit-identical to the direct loop below)
    float e[CH + 6];
#pragma unroll
    for (int i = 0; i < CH + 6; ++i) {
      const int t = t0 - 3 + i;
      e[i] = (t >= 0 && t < T) ? sS[pidx(t)] : -INFINITY;
    }
#pragma unroll
    for (int i = 0; i < CH + 5; ++i) e[i] = fmaxf(e[i], e[i + 1]);       // e[i..i+1]
#pragma unroll
    for (int i = 0; i < CH + 3; ++i) e[i] = fmaxf(e[i], e[i + 2]);       // e[i..i+3]
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int t = t0 + i;
      float v = fmaxf(e[i], e[i + 3]);                                    // e[i..i+6] = t-3..t+3
      if (t >= T - c.w) v = __int_as_float(0x7f800000);  // +inf: the observation window is always kept
      else if (red) v -= rscale * expf((rr[t] - rmax) * inv_tau);
      key[i] = t < T ? orderable(v) : 0u;
    }
  } else {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int t = t0 + i;
      float v = 0.f;
      if (t < T) {
        if (t >= T - c.w) {
          v = __int_as_float(0x7f800000);            // +inf: the observation window is always kept
        } else {
          v = sS[pidx(t)];
          const int lo = max(0, t - half), hi = min(T - 1, t + half);
          for (int j = lo; j <= hi; ++j) v = fmaxf(v, sS[pidx(j)]);
          if (red) v -= rscale * expf((rr[t] - rmax) * inv_tau);
        }
      }
      key[i] = t < T ? orderable(v) : 0u;            // 0 = below every real key; never selected (ell <= T)
    }
  }

  // MSB radix select of the ell-th largest key (as k_select)
  const int lane = threadIdx.x & 31;
  uint32_t mask = 0;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const bool in = t0 + i < T && (key[i] & mask) == prefix;
      const uint32_t d = (key[i] >> shift) & 255u;
      // a plain predicated increment: sm_100a merges the lanes of one instruction that hit the same
      // address (ATOMS.POPC.INC). Measured (select ms, qwen7b / llama8b / qwen32b): a software
      // whole-warp-one-digit path (ballot + shfl + all) 0.47 / 0.92 / 2.02, this 0.31 / 0.59 / 1.40;
      // three 11-bit passes (2048 bins, block scan) 0.34 / 0.59 / 1.34
      if (in) atomicAdd(&hist[d], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      int cnt[8];
      int sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { cnt[i] = hist[255 - (lane * 8 + i)]; sum += cnt[i]; }
      const int incl = warp_incl_scan(sum);
      const int excl = incl - sum;
      const int need = s_need;
      int found = -1, above = 0, run = excl;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (found < 0 && run < need && run + cnt[i] >= need) { found = 255 - (lane * 8 + i); above = run; }
        run += cnt[i];
      }
      const unsigned ball = __ballot_sync(0xffffffffu, found >= 0);
      const int src = __ffs(ball) - 1;
      const int d = __shfl_sync(0xffffffffu, found, src);
      const int ab = __shfl_sync(0xffffffffu, above, src);
      if (lane == 0) { s_prefix = prefix | ((uint32_t)d << shift); s_need = need - ab; }
    }
    mask |= 0xffu << shift;
    __syncthreads();
  }
  const uint32_t kstar = s_prefix;
  const int need_eq = s_need;

  // emission (as k_select): equal keys kept latest-first, kept positions written ascending
  int eq = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) eq += (t0 + i < T && key[i] == kstar);
  int eq_tot;
  const int eq_before = block_excl_t<NT>(eq, sm, &eq_tot);
  int eq_after = eq_tot - eq_before - eq;
  uint32_t keepm = 0;
  int kept_here = 0;
#pragma unroll
  for (int i = CH - 1; i >= 0; --i) {
    bool keep = false;
    if (t0 + i < T) {
      keep = key[i] > kstar;
      if (key[i] == kstar) { keep = eq_after < need_eq; ++eq_after; }
    }
    keepm |= (uint32_t)keep << i;
    kept_here += keep;
  }
  int kept_tot;
  const int out0 = block_excl_t<NT>(kept_here, sm, &kept_tot);
  int32_t* out = c.ws.kept + (size_t)unit * c.ws.kept_stride;
  int o = out0;
#pragma unroll
  for (int i = 0; i < CH; ++i)
    if (keepm >> i & 1u) { ZPC_CHECK(o < ell && t0 + i < T); out[o++] = t0 + i; }
}

template <int NT, int CH>
__global__ void __launch_bounds__(NT, NT == 256 ? 3 : (NT == 512 ? 2 : 1)) k_select_reg(Call c) {
  if (*c.status != ZPC_OK) return;
  select_reg_unit<NT, CH>(c, blockIdx.x);
}

}  // namespace

cudaError_t launch_select(const Call& c, cudaStream_t s) {
  const int units = c.R * c.L * c.h_kv;
  if (units == 0) return cudaSuccess;
  // register-resident variant while a thread's chunk fits CH <= 32 keys. params.variant (tests and A/B
  // runs): select 1 = always k_select, 2 = k_select_reg for every T <= 32K, 0 = by T as below
  const int vsel = (int)((c.variant >> ZPC_V_SELECT_SHIFT) & 3u);
  const int mode = vsel == 0 ? 1 : (vsel == 1 ? 0 : 2);
  const bool reg = mode != 0;
  const int T = c.max_seq_len;
  // T <= 4K (the paper's operating point, T = 2304): k_select_reg<256, 16> when there are >= 4 units per SM
  // (paper_op, 4 requests, 1152 units: 0.041 ms vs 0.045 for k_select), k_select below that (1 request, 288
  // units: 0.017 vs 0.019 -- 1024-thread CTAs spread a small call over more of the SMs)
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return cudaErrorInvalidDevice;
  const bool many = units >= 4 * sms;
  if (reg && (T > 4 * kThreads || mode == 2 || many) && T <= 32 * kThreads) {
    const size_t smem = sizeof(float) * (size_t)(T + T / 32 + 1);
    auto launch = [&](auto kern, int nt) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<units, nt, smem, s>>>(c);
      return cudaGetLastError();
    };
    // 32 keys per thread and a CTA that shrinks with T, so 8K units run 3 CTAs per SM; 16 keys for T <= 4K
    if (T <= 16 * 256) return launch(k_select_reg<256, 16>, 256);
    if (T <= 32 * 256) return launch(k_select_reg<256, 32>, 256);
    if (T <= 32 * 512) return launch(k_select_reg<512, 32>, 512);
    return launch(k_select_reg<1024, 32>, 1024);
  }
  if (c.max_seq_len > kSelectSmemMaxT) {   // keys in the workspace (select_keys region)
    k_select<true><<<units, kThreads, 0, s>>>(c);
    return cudaGetLastError();
  }
  const size_t smem = sizeof(uint32_t) * (size_t)c.max_seq_len;
  cudaFuncSetAttribute(k_select<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_select<false><<<units, kThreads, smem, s>>>(c);
  return cudaGetLastError();
}

}  // namespace zpc
