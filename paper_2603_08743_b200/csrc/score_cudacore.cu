// a1 + a2 on CUDA cores (FFMA): the fp32-pool path (the toy config; tf32 tensor cores would
// break the 1e-3 tolerance) and the reference fallback for bf16 when the
// tcgen05 kernel is disabled by ZPC_F_SCORE_CUDACORE.
//
// Two passes (with ZPC_F_LSE_INPUT pass 1 is replaced by k_lse_input):
//   pass 1 (k_lse_cc, one CTA per unit, one thread per window column c = u*G + g):
//          LSE2[c] = log2 sum_{t <= T-w+u} 2^{x2[c,t]},  x2 = (q.k) * log2(e)/sqrt(d)
//   pass 2 (k_final_cc, one thread per token):
//          S[t] = (1/w) sum_{u: t <= T-w+u} 2^{max_g (x2[(u,g),t] - LSE2[(u,g)])}
//   which is the mean over u of the max over g of softmax: exp is monotone,
//   so max_g exp(a_g) = exp(max_g a_g) and the max is taken before the exponential.
#include "internal.h"

namespace zpc {
namespace {

constexpr int kLseThreads = 256;   // >= G*w (host checks G*w <= 256)
constexpr int kLseTile = 32;       // tokens staged per step
constexpr int kFinThreads = 128;   // tokens per CTA in pass 2

template <typename E>
__device__ __forceinline__ float ld_elem(const E* p, size_t i);
template <>
__device__ __forceinline__ float ld_elem<uint16_t>(const uint16_t* p, size_t i) { return bf16_to_f32(p[i]); }
template <>
__device__ __forceinline__ float ld_elem<float>(const float* p, size_t i) { return p[i]; }

template <typename E, int D>
__global__ void __launch_bounds__(kLseThreads) k_lse_cc(Call c) {
  if (*c.status != ZPC_OK) return;
  __shared__ float ks[kLseTile][D];
  const int unit = blockIdx.x;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int slot = c.q_slots[r];
  const int GW = c.G * c.w;
  const int col = threadIdx.x;
  const bool active = col < GW;
  const int u = active ? col / c.G : 0, g = active ? col % c.G : 0;
  const float scale = 1.4426950408889634f * rsqrtf((float)D);
  const E* Q = reinterpret_cast<const E*>(c.q_cache);
  const E* K = reinterpret_cast<const E*>(c.k_cache);
  const int* table = c.tables + (size_t)r * c.table_stride;
  float q[D];
  {
    const size_t qo = q_row(c, l, slot, u, h * c.G + g);
#pragma unroll
    for (int i = 0; i < D; ++i) q[i] = active ? ld_elem(Q, qo + i) * scale : 0.f;
  }
  const int limit = T - c.w + u;     // causal: window row u sits at position T-w+u (R1, R2)
  float m = -INFINITY, s = 0.f;
  for (int t0 = 0; t0 < T; t0 += kLseTile) {
    for (int e = threadIdx.x; e < kLseTile * D; e += kLseThreads) {
      const int tt = e / D, i = e % D, t = t0 + tt;
      ks[tt][i] = (t < T) ? ld_elem(K, kv_row(c, l, table[t / c.b], t % c.b, h) + i) : 0.f;
    }
    __syncthreads();
    const int n = min(kLseTile, T - t0);
    for (int tt = 0; tt < n; ++tt) {
      if (t0 + tt > limit) break;
      float x = 0.f;
#pragma unroll
      for (int i = 0; i < D; i += 4) {
        const float4 kv = *reinterpret_cast<const float4*>(&ks[tt][i]);
        x = fmaf(q[i], kv.x, x); x = fmaf(q[i + 1], kv.y, x);
        x = fmaf(q[i + 2], kv.z, x); x = fmaf(q[i + 3], kv.w, x);
      }
      if (x > m) { s = s * ex2f(m - x) + 1.f; m = x; }
      else s += ex2f(x - m);
    }
    __syncthreads();
  }
  if (active) c.ws.lse[(size_t)unit * GW + col] = m + lg2f(s);
}

// NEXT-4 (ZPC_F_LSE_INPUT): the normalisers come from the caller (the decode attention of each
// window position), so pass 1 is a relayout: LSE2[unit][u*G + g] = log2(e) * lse_in[l][slot][u][h*G + g].
__global__ void __launch_bounds__(kLseThreads) k_lse_input(Call c) {
  if (*c.status != ZPC_OK) return;
  const int unit = blockIdx.x;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int slot = c.q_slots[r];
  const int GW = c.G * c.w;
  for (int col = threadIdx.x; col < GW; col += kLseThreads) {
    const int u = col / c.G, g = col % c.G;
    const size_t at = (((size_t)l * c.M + slot) * c.w + u) * c.h_q + (size_t)h * c.G + g;
    c.ws.lse[(size_t)unit * GW + col] = c.lse_in[at] * 1.4426950408889634f;
  }
}

template <typename E, int D>
__global__ void __launch_bounds__(kFinThreads) k_final_cc(Call c) {
  if (*c.status != ZPC_OK) return;
  extern __shared__ float qs[];      // [GW][D] pre-scaled queries, then [GW] LSE2
  const int unit = blockIdx.y;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int t0 = blockIdx.x * kFinThreads;
  if (t0 >= T) return;
  const int slot = c.q_slots[r];
  const int GW = c.G * c.w;
  float* lse = qs + (size_t)GW * D;
  const float scale = 1.4426950408889634f * rsqrtf((float)D);
  const E* Q = reinterpret_cast<const E*>(c.q_cache);
  const E* K = reinterpret_cast<const E*>(c.k_cache);
  for (int e = threadIdx.x; e < GW * D; e += kFinThreads) {
    const int col = e / D, i = e % D;
    const int u = col / c.G, g = col % c.G;
    qs[e] = ld_elem(Q, q_row(c, l, slot, u, h * c.G + g) + i) * scale;
  }
  for (int e = threadIdx.x; e < GW; e += kFinThreads) lse[e] = c.ws.lse[(size_t)unit * GW + e];
  __syncthreads();
  const int t = t0 + threadIdx.x;
  if (t >= T) return;
  const int* table = c.tables + (size_t)r * c.table_stride;
  float k[D];
  const size_t ko = kv_row(c, l, table[t / c.b], t % c.b, h);
#pragma unroll
  for (int i = 0; i < D; ++i) k[i] = ld_elem(K, ko + i);
  float s = 0.f;
  for (int u = 0; u < c.w; ++u) {
    if (t > T - c.w + u) continue;       // masked for this window row
    float m = -INFINITY;
    for (int g = 0; g < c.G; ++g) {
      const int col = u * c.G + g;
      const float* qv = qs + (size_t)col * D;
      float x = 0.f;
#pragma unroll
      for (int i = 0; i < D; i += 4) {
        const float4 q4 = *reinterpret_cast<const float4*>(qv + i);
        x = fmaf(q4.x, k[i], x); x = fmaf(q4.y, k[i + 1], x);
        x = fmaf(q4.z, k[i + 2], x); x = fmaf(q4.w, k[i + 3], x);
      }
      m = fmaxf(m, x - lse[col]);
    }
    s += ex2f(m);
  }
  c.ws.scores[(size_t)unit * c.max_seq_len + t] = s / (float)c.w;
}

template <typename E, int D>
cudaError_t launch_typed(const Call& c, cudaStream_t s) {
  const int units = c.R * c.L * c.h_kv;
  if (units == 0) return cudaSuccess;
  if (c.lse_in) k_lse_input<<<units, kLseThreads, 0, s>>>(c);
  else k_lse_cc<E, D><<<units, kLseThreads, 0, s>>>(c);
  const size_t smem = sizeof(float) * ((size_t)c.G * c.w * D + (size_t)c.G * c.w);
  cudaFuncSetAttribute(k_final_cc<E, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((c.max_seq_len + kFinThreads - 1) / kFinThreads, units);
  k_final_cc<E, D><<<grid, kFinThreads, smem, s>>>(c);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_score_cudacore(const Call& c, cudaStream_t s) {
  if (c.dtype == ZPC_BF16) return c.d == 64 ? launch_typed<uint16_t, 64>(c, s) : launch_typed<uint16_t, 128>(c, s);
  return c.d == 64 ? launch_typed<float, 64>(c, s) : launch_typed<float, 128>(c, s);
}

}  // namespace zpc
