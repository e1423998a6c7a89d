// NEXT-1: lightning redundancy score (§C.7), per unit (r, l, h) and block of b
// tokens: C = cosine similarity of the block's key rows; C[i][i] = 0; per column j the LAST row i
// (newest token) with C[i][j] > p is zeroed ("we prioritize retaining newer tokens");
// r[t] = (row sum of C) / T. The softmax over the sequence with temperature tau and the combine
// S - lambda*R happen in k_select. Slots >= T take no part (R20); a zero-norm
// key has cosine 0 (R23); "above" is strictly greater (R21).
//
// k_red_mma (bf16, b = 16): one warp per block. The 16 rows are staged in shared memory (row stride
// padded by 16 B so ldmatrix is conflict-free) and the 16 x 16 Gram matrix is 2 x d/16
// mma.sync.m16n8k16 (bf16 -> fp32): one ldmatrix.x4 per K-step yields the A fragment and, because
// B is the block's own rows, both B fragments (n-tile 0 = {a0, a2}, n-tile 1 = {a1, a3}).
// k_red_generic (any dtype, b <= 32): one lane per row, fp32 dot products from L1; small/test shapes.
// k_red_tile (bf16, b = 32..256 in steps of 16, e.g. the paper's b = 256): one 256-thread CTA per
// block. The b rows are staged once in shared memory by cp.async (rows >= T zero-filled), each warp
// forms a pair of 16-row stripes of the b x b Gram matrix with ldmatrix + mma.sync.m16n8k16 (A
// fragments of both stripes held in registers across all column chunks, so each B fragment feeds
// four MMAs), and a single pass yields both results: the
// row sums of C over every column j != i, and per column the last row above p together with its
// value, packed (row + 1) << 32 | value into one 64-bit shared atomicMax (rows are unique within a
// column, so the maximum carries the value of the largest row). The zeroed entries are subtracted
// afterwards in ascending column order by the row's own thread (deterministic).
#include "internal.h"

namespace zpc {
namespace {

constexpr int kWarps = 8;            // warps per CTA (k_red_mma)
#ifndef ZPC_RED_BPW
// consecutive blocks per warp (the next block's rows are prefetched into registers while the current one is
// computed; the warp's block ids are read once). qwen7b --redundancy, k_red_mma ms at 8 / 16 / 32: 2.69 / 2.62 /
// 2.59 (0.87 / 0.89 / 0.90 of HBM): fewer warp prologues (first fetch not overlapped)
#define ZPC_RED_BPW 32
#endif
constexpr int kBlocksPerWarp = ZPC_RED_BPW;

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int D>
__global__ void __launch_bounds__(kWarps * 32) k_red_mma(Call c) {
  if (*c.status != ZPC_OK) return;
  constexpr int ROWB = D * 2 + 16;                 // padded row stride in shared memory (bytes)
  __shared__ __align__(16) uint8_t stage[kWarps][16 * ROWB];
  __shared__ float inv_norm[kWarps][16];
  const int unit = blockIdx.x;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int nb = (T + 15) / 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* table = c.tables + (size_t)r * c.table_stride;
  const uint16_t* K = reinterpret_cast<const uint16_t*>(c.k_cache);
  float* out = c.ws.redund + (size_t)unit * c.max_seq_len;
  const float inv_T = 1.0f / (float)T;
  const float p = c.red_p;
  uint8_t* st = stage[warp];
  const uint32_t st_s = (uint32_t)__cvta_generic_to_shared(st);
  const int r1 = lane >> 2, r2 = r1 + 8, cq = lane & 3;
  const int cols[4] = {2 * cq, 2 * cq + 1, 8 + 2 * cq, 9 + 2 * cq};

  constexpr int CPR = D / 8;                        // 16-B chunks per row
  constexpr int NV = 16 * CPR / 32;                 // 16-B vectors per lane per block
  const int jb_first = (blockIdx.y * kWarps + warp) * kBlocksPerWarp;
  int4 pre[NV];
  // the warp's block ids in one read (lane k holds block jb_first + k), so no fetch waits on a table read
  static_assert(kBlocksPerWarp <= 32, "one block id per lane");
  const int myblk = (lane < kBlocksPerWarp && jb_first + lane < nb) ? table[jb_first + lane] : 0;
  auto fetch = [&](int jb) {                        // this lane's share of block jb's 16 rows
    const int blk = __shfl_sync(0xffffffffu, myblk, jb - jb_first);
    ZPC_CHECK(blk >= 0 && blk < c.N_total);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int q = lane + 32 * v, row = q / CPR, ch = q % CPR;
      pre[v] = *reinterpret_cast<const int4*>(K + kv_row(c, l, blk, row, h) + ch * 8);
    }
  };
  if (jb_first < nb) fetch(jb_first);
  for (int k = 0; k < kBlocksPerWarp; ++k) {
    const int jb = jb_first + k;
    if (jb >= nb) break;
    const int j0 = jb * 16;
    const int nvalid = min(16, T - j0);
    // stage block jb (rows >= nvalid are loaded but masked), then start fetching block jb + 1
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int q = lane + 32 * v, row = q / CPR, ch = q % CPR;
      // slots >= T are zeroed, not just masked: a stale slot holding Inf/NaN would make 0 * NaN = NaN
      *reinterpret_cast<int4*>(st + row * ROWB + ch * 16) = row < nvalid ? pre[v] : make_int4(0, 0, 0, 0);
    }
    __syncwarp();
    if (k + 1 < kBlocksPerWarp && jb + 1 < nb) fetch(jb + 1);
    // Gram matrix G = K_blk K_blk^T (16 x 16, fp32), two n-tiles of 8 columns
    float g0[4] = {0.f, 0.f, 0.f, 0.f}, g1[4] = {0.f, 0.f, 0.f, 0.f};
    const uint32_t a_addr = st_s + (uint32_t)((lane & 15) * ROWB + (lane >> 4) * 16);
#pragma unroll
    for (int s = 0; s < D / 16; ++s) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(a_addr + s * 32, a0, a1, a2, a3);
      mma_bf16(g0, a0, a1, a2, a3, a0, a2);        // columns 0..7  (tokens 0..7)
      mma_bf16(g1, a0, a1, a2, a3, a1, a3);        // columns 8..15 (tokens 8..15)
    }
    // this thread: G[r1][cols[0..3]] = g0[0], g0[1], g1[0], g1[1]; G[r2][...] = g0[2], g0[3], g1[2], g1[3]
    float v1[4] = {g0[0], g0[1], g1[0], g1[1]}, v2[4] = {g0[2], g0[3], g1[2], g1[3]};
    // squared norms from the diagonal -> 1/norm (0 for a zero-norm key or an invalid slot)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (cols[e] == r1) inv_norm[warp][r1] = (v1[e] > 0.f && r1 < nvalid) ? 1.0f / sqrtf(v1[e]) : 0.f;
      if (cols[e] == r2) inv_norm[warp][r2] = (v2[e] > 0.f && r2 < nvalid) ? 1.0f / sqrtf(v2[e]) : 0.f;
    }
    __syncwarp();
    const float n1 = inv_norm[warp][r1], n2 = inv_norm[warp][r2];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float nc = inv_norm[warp][cols[e]];
      v1[e] = (cols[e] == r1) ? 0.f : v1[e] * n1 * nc;   // invalid rows/cols carry a 0 norm
      v2[e] = (cols[e] == r2) ? 0.f : v2[e] * n2 * nc;
      // the column's last (largest row index) entry above p: rows of this column are spread over
      // the 8 threads with the same lane & 3 (each holds rows r1 and r2 = r1 + 8)
      int cand = v2[e] > p ? r2 : (v1[e] > p ? r1 : -1);
      cand = max(cand, __shfl_xor_sync(0xffffffffu, cand, 4));
      cand = max(cand, __shfl_xor_sync(0xffffffffu, cand, 8));
      cand = max(cand, __shfl_xor_sync(0xffffffffu, cand, 16));
      if (cand == r1) v1[e] = 0.f;
      if (cand == r2) v2[e] = 0.f;
    }
    float s1 = (v1[0] + v1[1]) + (v1[2] + v1[3]);
    float s2 = (v2[0] + v2[1]) + (v2[2] + v2[3]);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
    s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
    if (cq == 0) {
      if (r1 < nvalid) out[j0 + r1] = s1 * inv_T;
      if (r2 < nvalid) out[j0 + r2] = s2 * inv_T;
    }
    __syncwarp();   // the stage and inv_norm are rewritten for the next block
  }
}

// any dtype, b <= 32: lane i owns row i of the block
__global__ void __launch_bounds__(kWarps * 32) k_red_generic(Call c) {
  if (*c.status != ZPC_OK) return;
  const int unit = blockIdx.x;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int b = c.b;
  const int nb = (T + b - 1) / b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* table = c.tables + (size_t)r * c.table_stride;
  float* out = c.ws.redund + (size_t)unit * c.max_seq_len;
  const float inv_T = 1.0f / (float)T;
  for (int jb = blockIdx.y * kWarps + warp; jb < nb; jb += gridDim.y * kWarps) {
    const int j0 = jb * b;
    const int nvalid = min(b, T - j0);
    const int blk = table[jb];
    ZPC_CHECK(blk >= 0 && blk < c.N_total);
    const bool mine = lane < nvalid;
    auto elem = [&](int row, int e) -> float {
      const size_t off = kv_row(c, l, blk, row, h) + e;
      return c.dtype == ZPC_BF16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(c.k_cache)[off])
                                 : reinterpret_cast<const float*>(c.k_cache)[off];
    };
    float dots[32];
    float nrm2 = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) dots[j] = 0.f;
    if (mine) {
      for (int e = 0; e < c.d; ++e) {
        const float ki = elem(lane, e);
        nrm2 = fmaf(ki, ki, nrm2);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nvalid) dots[j] = fmaf(ki, elem(j, e), dots[j]);
      }
    }
    const float inv_n = (mine && nrm2 > 0.f) ? 1.0f / sqrtf(nrm2) : 0.f;
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j >= b) break;
      const float inv_nj = __shfl_sync(0xffffffffu, inv_n, j);
      float cij = (mine && j < nvalid && j != lane) ? dots[j] * inv_n * inv_nj : 0.f;
      int cand = cij > c.red_p ? lane : -1;
#pragma unroll
      for (int o = 16; o; o >>= 1) cand = max(cand, __shfl_xor_sync(0xffffffffu, cand, o));
      if (cand == lane) cij = 0.f;
      sum += cij;
    }
    if (mine) out[j0 + lane] = sum * inv_T;
  }
}

constexpr int kTileThreads = 256;

template <int D>
__host__ __device__ constexpr int tile_rowb() { return D * 2 + 16; }   // padded row stride (bytes)

inline size_t tile_smem_bytes(int D, int b) {
  return (size_t)b * (D * 2 + 16) + (size_t)b * (sizeof(float) * 2 + sizeof(unsigned long long)) +
         (size_t)(b / 16) * b * sizeof(float);
}

template <int D>
__global__ void __launch_bounds__(kTileThreads) k_red_tile(Call c) {
  if (*c.status != ZPC_OK) return;
  constexpr int ROWB = tile_rowb<D>();
  constexpr int CPR = D / 8;                        // 16-B chunks per row
  extern __shared__ __align__(16) uint8_t smem[];
  const int b = c.b;
  uint8_t* st = smem;
  unsigned long long* last = reinterpret_cast<unsigned long long*>(smem + (size_t)b * ROWB);
  float* inv_norm = reinterpret_cast<float*>(last + b);
  float* rowsum = inv_norm + b;
  float* colpart = rowsum + b;                       // [b/16][b] column sums of mirrored tiles
  const int unit = blockIdx.x;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int jb = blockIdx.y;
  if (jb * b >= T) return;
  const int j0 = jb * b;
  const int nvalid = min(b, T - j0);
  const int blk = c.tables[(size_t)r * c.table_stride + jb];
  ZPC_CHECK(blk >= 0 && blk < c.N_total);
  const uint16_t* K = reinterpret_cast<const uint16_t*>(c.k_cache);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // stage the block's rows by 16-B cp.async (16 threads per 256-B row, every copy in flight at once);
  // slots >= T are zero-filled (src-size 0, R20)
  const uint32_t st_s = (uint32_t)__cvta_generic_to_shared(st);
  for (int q = tid; q < b * CPR; q += kTileThreads) {
    const int row = q / CPR, ch = q % CPR;
    const bool ok = row < nvalid;
    const uint16_t* src = K + kv_row(c, l, blk, ok ? row : 0, h) + ch * 8;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(st_s + (uint32_t)(row * ROWB + ch * 16)),
                 "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int j = tid; j < b; j += kTileThreads) last[j] = 0ull;
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // 1/||k_i|| in fp32 (0 for a zero-norm key or an empty slot, R23)
  for (int i = tid; i < b; i += kTileThreads) {
    float s = 0.f;
#pragma unroll
    for (int ch = 0; ch < CPR; ++ch) {
      const uint4 v = *reinterpret_cast<const uint4*>(st + i * ROWB + ch * 16);
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float lo = __uint_as_float(w4[e] << 16), hi = __uint_as_float(w4[e] & 0xffff0000u);
        s = fmaf(lo, lo, s);
        s = fmaf(hi, hi, s);
      }
    }
    inv_norm[i] = s > 0.f ? 1.0f / sqrtf(s) : 0.f;
  }
  __syncthreads();

  const float p = c.red_p;
  const uint32_t frag_off = (uint32_t)((lane & 15) * ROWB + (lane >> 4) * 16);
  const int cq = lane & 3;
  // C is symmetric: only the tiles (stripe m, column group n >= m) of 16 x 16 are formed. Warp w owns
  // stripes w and MT-1-w (MT + 1 tiles per warp for even MT): for n >= MT-1-w one ldmatrix B fragment
  // feeds both stripes' MMAs. An off-diagonal tile (n > m) also stands for its mirror (n, m): its
  // column sums go to colpart[m][j] (summed in ascending m at the end, deterministic) and each row's
  // last column above p is a candidate for the column i = that row.
  const int MT = b / 16;
  for (int w2 = warp; 2 * w2 < MT; w2 += kTileThreads / 32) {
    const int ms[2] = {w2, MT - 1 - w2};
    const bool two = ms[1] != ms[0];                 // warp-uniform: a distinct second stripe
    int rr[2][2];
    float nn[2][2], rs[2][2];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      rr[m][0] = ms[m] * 16 + (lane >> 2);
      rr[m][1] = rr[m][0] + 8;
      nn[m][0] = inv_norm[rr[m][0]];
      nn[m][1] = inv_norm[rr[m][1]];
      rs[m][0] = rs[m][1] = 0.f;
    }
    uint32_t a[2][D / 16][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int s = 0; s < D / 16; ++s)
        ldsm_x4(st_s + (uint32_t)(ms[m] * 16 * ROWB) + frag_off + s * 32, a[m][s][0], a[m][s][1], a[m][s][2],
                a[m][s][3]);
    for (int n = ms[0]; n < MT; ++n) {               // column group n: columns 16n .. 16n+15
      const bool useB = two && n >= ms[1];
      float acc[2][2][4];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int q = 0; q < 2; ++q) acc[m][q][0] = acc[m][q][1] = acc[m][q][2] = acc[m][q][3] = 0.f;
#pragma unroll
      for (int s = 0; s < D / 16; ++s) {
        uint32_t x0, x1, x2, x3;
        ldsm_x4(st_s + (uint32_t)(n * 16 * ROWB) + frag_off + s * 32, x0, x1, x2, x3);
        mma_bf16(acc[0][0], a[0][s][0], a[0][s][1], a[0][s][2], a[0][s][3], x0, x2);      // +0..7
        mma_bf16(acc[0][1], a[0][s][0], a[0][s][1], a[0][s][2], a[0][s][3], x1, x3);      // +8..15
        if (useB) {
          mma_bf16(acc[1][0], a[1][s][0], a[1][s][1], a[1][s][2], a[1][s][3], x0, x2);
          mma_bf16(acc[1][1], a[1][s][0], a[1][s][1], a[1][s][2], a[1][s][3], x1, x3);
        }
      }
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        if (m == 1 && !useB) continue;
        const int r1 = rr[m][0], r2 = rr[m][1];
        const bool mirror = n > ms[m];               // warp-uniform
        // this lane's 4 columns jc(k) = 16n + (k >> 1) * 8 + 2 * (lane & 3) + (k & 1), rows r1 and r2
        float v1[4], v2[4];
        bool hit = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int j = n * 16 + (k >> 1) * 8 + 2 * cq + (k & 1);
          const float nj = inv_norm[j];
          v1[k] = (j == r1) ? 0.f : acc[m][k >> 1][k & 1] * nn[m][0] * nj;
          v2[k] = (j == r2) ? 0.f : acc[m][k >> 1][2 + (k & 1)] * nn[m][1] * nj;
          rs[m][0] += v1[k];
          rs[m][1] += v2[k];
          hit |= (v1[k] > p) | (v2[k] > p);
        }
        if (mirror) {
          // C[j][i] summed over the stripe's 16 rows i: the lane's 4 column partials reduced over the 8
          // lanes sharing lane & 3 by a halving butterfly (bits 4, 3, then 2 of the lane: 4 shuffles)
          float cs[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) cs[k] = v1[k] + v2[k];
          const bool h16 = lane & 16, h8 = lane & 8;
          const float k0 = (h16 ? cs[2] : cs[0]) + __shfl_xor_sync(0xffffffffu, h16 ? cs[0] : cs[2], 16);
          const float k1 = (h16 ? cs[3] : cs[1]) + __shfl_xor_sync(0xffffffffu, h16 ? cs[1] : cs[3], 16);
          float t = (h8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
          t += __shfl_xor_sync(0xffffffffu, t, 4);
          const int kk = (h16 ? 2 : 0) + (h8 ? 1 : 0);
          if (!(lane & 4)) colpart[ms[m] * b + n * 16 + (kk >> 1) * 8 + 2 * cq + (kk & 1)] = t;
        }
        // rare path (warp-uniform): some cosine of this tile is above p
        if (__any_sync(0xffffffffu, hit)) {
          unsigned long long kr1 = 0ull, kr2 = 0ull;  // rows' last column above p (mirror candidates)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int j = n * 16 + (k >> 1) * 8 + 2 * cq + (k & 1);
            if (mirror) {                            // columns ascend with k: the last one above p wins
              if (v1[k] > p) kr1 = ((unsigned long long)(j + 1) << 32) | __float_as_uint(v1[k]);
              if (v2[k] > p) kr2 = ((unsigned long long)(j + 1) << 32) | __float_as_uint(v2[k]);
            }
            // the stripe's last row above p in column j; the column's rows sit on the 8 lanes sharing
            // lane & 3
            unsigned long long key = v2[k] > p   ? ((unsigned long long)(r2 + 1) << 32) | __float_as_uint(v2[k])
                                     : v1[k] > p ? ((unsigned long long)(r1 + 1) << 32) | __float_as_uint(v1[k])
                                                 : 0ull;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
              const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
              key = other > key ? other : key;
            }
            if (lane < 4 && key) atomicMax(&last[j], key);
          }
          // mirror: column r's candidates are the rows j (> r) of group n, i.e. row r's columns, which
          // sit on the 4 lanes sharing lane >> 2
          if (mirror) {
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
              const unsigned long long o1 = __shfl_xor_sync(0xffffffffu, kr1, o);
              const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, kr2, o);
              kr1 = o1 > kr1 ? o1 : kr1;
              kr2 = o2 > kr2 ? o2 : kr2;
            }
            if (cq == 0 && kr1) atomicMax(&last[r1], kr1);
            if (cq == 0 && kr2) atomicMax(&last[r2], kr2);
          }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      if (m == 1 && !two) continue;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        float v = rs[m][k];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (cq == 0) rowsum[rr[m][k]] = v;
      }
    }
  }
  __syncthreads();
  // remove each column's zeroed entry from its row, in ascending column order; r[t] = sum / T
  float* out = c.ws.redund + (size_t)unit * c.max_seq_len;
  const float inv_T = 1.0f / (float)T;
  for (int i0 = warp * 32; i0 < b; i0 += kTileThreads) {
    const int i = i0 + lane;                         // b is a multiple of 16: i < b for lanes < 16
    float s = 0.f;
    if (i < b) {                                     // own-stripe tiles + mirrored tiles of stripes above
      s = rowsum[i];
      for (int m = 0; m < i / 16; ++m) s += colpart[m * b + i];
    }
    for (int jc = 0; jc < b; jc += 32) {             // columns with a zeroed entry, ascending
      const unsigned long long key = jc + lane < b ? last[jc + lane] : 0ull;
      uint32_t any = __ballot_sync(0xffffffffu, key != 0ull);
      while (any) {
        const int src = __ffs(any) - 1;
        any &= any - 1;
        const unsigned long long k = __shfl_sync(0xffffffffu, key, src);
        if ((int)(k >> 32) == i + 1) s -= __uint_as_float((uint32_t)k);
      }
    }
    if (i < nvalid) out[j0 + i] = s * inv_T;
  }
}

}  // namespace

cudaError_t launch_redundancy(const Call& c, cudaStream_t s) {
  const int units = c.R * c.L * c.h_kv;
  if (units == 0) return cudaSuccess;
  if (c.dtype == ZPC_BF16 && c.b == 16) {
    const int nb_max = (c.max_seq_len + 15) / 16;
    const dim3 grid(units, (nb_max + kWarps * kBlocksPerWarp - 1) / (kWarps * kBlocksPerWarp));
    if (c.d == 128) k_red_mma<128><<<grid, kWarps * 32, 0, s>>>(c);
    else k_red_mma<64><<<grid, kWarps * 32, 0, s>>>(c);
  } else if (c.dtype == ZPC_BF16 && c.b > 16 && c.b % 16 == 0 && c.b <= 256 && !(c.variant & ZPC_V_RED_MMASYNC)) {
    return launch_redundancy_tc(c, s);
  } else if (c.dtype == ZPC_BF16 && c.b > 16 && c.b % 16 == 0 && c.b <= 256) {
    const dim3 grid(units, (c.max_seq_len + c.b - 1) / c.b);
    const size_t smem = tile_smem_bytes(c.d, c.b);
    cudaError_t e;
    if (c.d == 128) {
      e = cudaFuncSetAttribute(k_red_tile<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      // 3 CTAs of b = 256 per SM need the whole carveout
      e = cudaFuncSetAttribute(k_red_tile<128>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return e;
      k_red_tile<128><<<grid, kTileThreads, smem, s>>>(c);
    } else {
      e = cudaFuncSetAttribute(k_red_tile<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(k_red_tile<64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return e;
      k_red_tile<64><<<grid, kTileThreads, smem, s>>>(c);
    }
  } else {
    const int nb_max = (c.max_seq_len + c.b - 1) / c.b;
    const dim3 grid(units, min(64, (nb_max + kWarps - 1) / kWarps));
    k_red_generic<<<grid, kWarps * 32, 0, s>>>(c);
  }
  return cudaGetLastError();
}

}  // namespace zpc
