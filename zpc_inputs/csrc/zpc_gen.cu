// Device twin of zpc_inputs/workloads.py: fills K/V pools and the Q window cache in HBM with
// bytes bit-identical to the numpy generator (all integer arithmetic + exact scaling + RNE).
// Input generation only — holds none of the compression method's arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

extern "C" {
typedef struct {
  int32_t L, h_kv, h_q, d, b, N_total, M, w, dtype;  // dtype 0 = bf16, 1 = fp32
  int32_t structured, prefix_tokens;
  uint64_t seed;
} zpcgen_cfg;
}

namespace {

constexpr uint32_t KIND_K = 1, KIND_V = 2, KIND_Q = 3, KIND_DIR = 4, KIND_ROLE = 5;
constexpr uint32_t PREFIX_RID = 0xFFFFFF;
constexpr int AMP_UNIT = 8192, Q_AMP = 2 * 8192, SINKS = 4, RECENT = 256;

struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

__device__ __forceinline__ uint32_t kindword(uint32_t kind, int l, int h) { return (kind << 24) | (l << 8) | h; }

__device__ __forceinline__ int z_of(uint32_t a, uint32_t b) {
  return (int)((a & 0xFFFF) + (a >> 16) + (b & 0xFFFF) + (b >> 16)) - 2 * 65535;
}

__device__ __forceinline__ int dir_of(const zpcgen_cfg& c, int l, int h, int i) {
  U4 r = philox((uint32_t)i, 0u, kindword(KIND_DIR, l, h), 0u, (uint32_t)c.seed, (uint32_t)(c.seed >> 32));
  return (r.x & 1) ? 1 : -1;
}

__device__ __forceinline__ int amp_of(const zpcgen_cfg& c, uint32_t rid, int l, int h, int pos, int T) {
  if (!c.structured) return 0;
  U4 r = philox((uint32_t)pos, rid, kindword(KIND_ROLE, l, h), 0u, (uint32_t)c.seed, (uint32_t)(c.seed >> 32));
  int amp = 0;
  if ((r.x & 0xFF) < 5) {
    const int cat = (r.x >> 8) & 3;
    amp = cat == 0 ? 3 : cat == 1 ? 4 : cat == 2 ? 5 : 4;
  }
  if (pos < SINKS) amp = 6;
  if (pos >= T - RECENT) amp = max(amp, 2);
  return amp;
}

__device__ __forceinline__ void store(const zpcgen_cfg& c, void* base, size_t idx, int xi) {
  const float f = (float)xi * 3.0517578125e-05f;  // 2^-15, exact
  if (c.dtype == 1) {
    reinterpret_cast<float*>(base)[idx] = f;
  } else {
    const uint32_t bits = __float_as_uint(f);
    reinterpret_cast<uint16_t*>(base)[idx] = (uint16_t)((bits + 0x7FFFu + ((bits >> 16) & 1u)) >> 16);
  }
}

// One thread per (request, layer, head, position, element pair).
__global__ void k_fill_kv(zpcgen_cfg c, void* K, void* V, const int32_t* tables, int32_t stride,
                          const int32_t* seq_lens, const int32_t* rids, int32_t R, int32_t T_max) {
  const int pairs = c.d / 2;
  const size_t total = (size_t)R * c.L * c.h_kv * T_max * pairs;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(g % pairs);
    size_t rest = g / pairs;
    const int pos = (int)(rest % T_max); rest /= T_max;
    const int h = (int)(rest % c.h_kv); rest /= c.h_kv;
    const int l = (int)(rest % c.L);
    const int r = (int)(rest / c.L);
    const int T = seq_lens[r];
    if (pos >= T) continue;
    const uint32_t rid = pos < c.prefix_tokens ? PREFIX_RID : (uint32_t)rids[r];
    const int blk = tables[(size_t)r * stride + pos / c.b];
    const size_t row = ((((size_t)l * c.N_total + blk) * c.b + pos % c.b) * c.h_kv + h) * (size_t)c.d;
    const uint32_t k0 = (uint32_t)c.seed, k1 = (uint32_t)(c.seed >> 32);
    U4 zk = philox((uint32_t)pos, rid, kindword(KIND_K, l, h), (uint32_t)i, k0, k1);
    U4 zv = philox((uint32_t)pos, rid, kindword(KIND_V, l, h), (uint32_t)i, k0, k1);
    const int amp = amp_of(c, rid, l, h, pos, T) * AMP_UNIT;
    const int ka = z_of(zk.x, zk.y) + amp * dir_of(c, l, h, 2 * i);
    const int kb = z_of(zk.z, zk.w) + amp * dir_of(c, l, h, 2 * i + 1);
    store(c, K, row + 2 * i, ka);
    store(c, K, row + 2 * i + 1, kb);
    store(c, V, row + 2 * i, z_of(zv.x, zv.y));
    store(c, V, row + 2 * i + 1, z_of(zv.z, zv.w));
  }
}

// One thread per (request, layer, window row, query head, element pair).
__global__ void k_fill_q(zpcgen_cfg c, void* Q, const int32_t* q_slots, const int32_t* rids, int32_t R) {
  const int pairs = c.d / 2;
  const int G = c.h_q / c.h_kv;
  const size_t total = (size_t)R * c.L * c.w * c.h_q * pairs;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(g % pairs);
    size_t rest = g / pairs;
    const int hq = (int)(rest % c.h_q); rest /= c.h_q;
    const int u = (int)(rest % c.w); rest /= c.w;
    const int l = (int)(rest % c.L);
    const int r = (int)(rest / c.L);
    U4 z = philox((uint32_t)u, (uint32_t)rids[r], kindword(KIND_Q, l, hq), (uint32_t)i, (uint32_t)c.seed,
                  (uint32_t)(c.seed >> 32));
    const int amp = c.structured ? Q_AMP : 0;
    const size_t row = ((((size_t)l * c.M + q_slots[r]) * c.w + u) * c.h_q + hq) * (size_t)c.d;
    store(c, Q, row + 2 * i, z_of(z.x, z.y) + amp * dir_of(c, l, hq / G, 2 * i));
    store(c, Q, row + 2 * i + 1, z_of(z.z, z.w) + amp * dir_of(c, l, hq / G, 2 * i + 1));
  }
}

}  // namespace

extern "C" {

int zpcgen_fill_kv(const zpcgen_cfg* c, void* K, void* V, const int32_t* tables, int32_t stride,
                   const int32_t* seq_lens, const int32_t* rids, int32_t R, int32_t T_max, void* stream) {
  if (R <= 0) return 0;
  k_fill_kv<<<148 * 16, 256, 0, static_cast<cudaStream_t>(stream)>>>(*c, K, V, tables, stride, seq_lens, rids, R,
                                                                      T_max);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int zpcgen_fill_q(const zpcgen_cfg* c, void* Q, const int32_t* q_slots, const int32_t* rids, int32_t R, void* stream) {
  if (R <= 0) return 0;
  k_fill_q<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(*c, Q, q_slots, rids, R);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}
