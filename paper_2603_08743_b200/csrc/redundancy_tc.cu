// NEXT-1 on 5th-generation tensor cores: the lightning redundancy score of one key block per CTA
// (PAPER.md:616-620 §C.7, :500-502; readings R19-R23 in DESIGN.md §2), for bf16 blocks of b = 32..256
// tokens (b % 16 == 0; the paper's operating point is b = 256).
//
// What it computes, per unit (r, l, h) and block of b tokens: C[i][j] = k_i.k_j / (|k_i| |k_j|),
// C[i][i] = 0; per column j the entry of the LAST row i (newest token) with C[i][j] > p is zeroed;
// r[t] = (row sum of C) / T. Slots >= T are zero rows (cosine 0, R20); a zero-norm key has cosine 0 (R23).
//
// How (k_red_umma): the block's rows are staged once in shared memory by 16-B cp.async, straight into the
// K-major 128-byte-swizzled UMMA layout; that one copy is both operands of the Gram matrix. Rows are cut
// into M = 128 halves: half m is ONE tcgen05.mma chain (M = 128 rows, N = b columns, d/16 K-steps), fp32
// accumulator in TMEM (lane = row i, column = j). The epilogue reads each row from TMEM (8 warps: a lane
// quarter x a column half each), scales by 1/|k_i| 1/|k_j|, and in one sweep yields the row sum over
// j != i and the row's last column above p. C is symmetric, so "column i's last row above p" is row i's
// last column above p (rare path, taken warp-uniformly when a chunk's maximum exceeds p); the zeroed entry
// belongs to that other row and is subtracted from its sum afterwards, in ascending column order
// (deterministic).
#include <algorithm>
#include <cstring>

#include "internal.h"
#include "tc_util.h"

namespace zpc {
namespace {

constexpr int kRThreads = 256;   // 8 warps: lane quarter (w & 3) x column half (w >> 2)

template <int D>
struct RedCfg {
  static constexpr int SLABS = D / 64;   // 64-element (128-B) K slabs
  static constexpr int KSTEPS = D / 16;
};

__host__ __device__ constexpr int red_rows(int b) { return b <= 128 ? 128 : 256; }   // A reads 128-row halves
// TMEM columns per CTA: one MMA covers at most 128 columns (a block of b > 128 is two column halves), so three
// CTAs fit an SM's 512 columns and no CTA waits in tcgen05.alloc
__host__ __device__ inline uint32_t red_tmem_cols(int b) { return b <= 32 ? 32u : b <= 64 ? 64u : 128u; }
inline size_t red_smem_bytes(int D, int b) {
  // operand rows + inv_norm, sq (zc, zv later), 2 x (row sum, last column, value) + bar, slot: <= 73.8 KB, so
  // three CTAs fit an SM
  return (size_t)red_rows(b) * D * 2 + (size_t)256 * 4 * 8 + 64;   // (2 barriers + TMEM slot in the last 64 B)
}

template <int D>
__global__ void __launch_bounds__(kRThreads, 3) k_red_umma(Call c, const __grid_constant__ CUtensorMap tmap_k, int ktma) {
  using C = RedCfg<D>;
  if (*c.status != ZPC_OK) return;
  const int unit = blockIdx.x;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int jb = blockIdx.y;
  if (jb * c.b >= T) return;
  const int b = c.b;
  const int rows = red_rows(b);
  const int j0 = jb * b;
  const int nvalid = min(b, T - j0);
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();     // SW128 operands need the 1024-B aligned base
  const uint32_t slab_bytes = (uint32_t)rows * 128u;
  float* inv_norm = reinterpret_cast<float*>(smem + (size_t)rows * D * 2);
  float* sq = inv_norm + 256;                       // [256] |k_i|^2 (fp32)
  float* rsum = sq + 256;                           // [2][256] row sums per column-split warp
  int* zpart = reinterpret_cast<int*>(rsum + 512);  // [2][256] last column above p (-1: none)
  float* zvpart = reinterpret_cast<float*>(zpart + 512);
  int* zc = reinterpret_cast<int*>(inv_norm);      // [256] per column i: the row whose entry (row, i) is zeroed
  float* zv = sq;                                   //        and that entry's value (both after the epilogues)
  uint64_t* bar = reinterpret_cast<uint64_t*>(zvpart + 512);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);   // bar[0] MMA, bar[1] TMA load
  int* zflag = reinterpret_cast<int*>(tmem_slot + 1);           // some entry of the block is above p
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t base = smem_u32(smem);
  const uint32_t ncols = red_tmem_cols(b);

  const int blk = c.tables[(size_t)r * c.table_stride + jb];
  ZPC_CHECK(blk >= 0 && blk < c.N_total);
  const uint32_t lbar = smem_u32(bar + 1);         // TMA load barrier (ktma)
  if (ktma) {
    // the block's b rows of head h: one TMA box of b slots x 64 elements per slab (row stride h_kv*d), landing in
    // the SW128 K-major layout; slots >= T are zeroed after it lands (R20)
    if (tid == 0) {
      mbar_init(lbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(lbar, (uint32_t)(b * D * 2));
      for (int sl = 0; sl < C::SLABS; ++sl)
        tma_load_3d(base + (uint32_t)sl * slab_bytes, &tmap_k, sl * 64, h, (l * c.N_total + blk) * b, lbar,
                    policy_evict_first());
    }
  } else {
    // ---- stage rows [0, rows) by 16-B cp.async into SW128 K-major slabs; rows >= nvalid are zero (R20).
    // Thread t copies 16-B chunk t % CPR of rows t / CPR + k * RPP: constant source / destination strides, and
    // the swizzle term is fixed because RPP is a multiple of 8.
    constexpr int CPR = D / 8;                      // 16-B chunks per row
    constexpr int RPP = kRThreads / CPR;            // rows per pass (16 or 32)
    static_assert(RPP % 8 == 0, "swizzle phase must repeat every pass");
    const int ch = tid % CPR, row0 = tid / CPR;
    const size_t hD = (size_t)c.h_kv * D;
    const uint16_t* src = reinterpret_cast<const uint16_t*>(c.k_cache) + kv_row(c, l, blk, 0, h) + ch * 8 +
                          (size_t)row0 * hD;
    uint32_t dst = base + (uint32_t)(ch >> 3) * slab_bytes + (uint32_t)row0 * 128u +
                   (uint32_t)(((ch & 7) ^ (row0 & 7)) << 4);
    for (int row = row0; row < rows; row += RPP, src += RPP * hD, dst += RPP * 128u) {
      const bool ok = row < nvalid;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(ok ? src : c.k_cache),
                   "r"(ok ? 16 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    *zflag = 0;
    mbar_init(smem_u32(bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (ktma) {
    __syncthreads();                                // lbar initialised before anyone waits on it
    // one warp polls the barrier; the others block in bar.sync (no issue slots spent spinning)
    if (warp == 0) mbar_wait_lean(lbar, 0);
    __syncthreads();
    if (nvalid < b) {                               // slots >= T of a partial last block: zero rows (R20)
      for (int q = tid; q < (b - nvalid) * (D / 8); q += kRThreads) {
        const int row = nvalid + q / (D / 8), ch = q % (D / 8);
        *reinterpret_cast<uint4*>(smem + (ch >> 3) * slab_bytes + row * 128 + (((ch & 7) ^ (row & 7)) << 4)) =
            make_uint4(0u, 0u, 0u, 0u);
      }
    }
  } else {
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  // |k_i|^2 and 1/|k_i| in fp32 (0 for a zero-norm key or an empty slot, R23)
  if (tid < b) {
    const int i = tid;
    uint64_t s2 = 0ull;
#pragma unroll
    for (int ch = 0; ch < D / 8; ++ch) {
      const uint4 v = *reinterpret_cast<const uint4*>(smem + (ch >> 3) * slab_bytes + i * 128 + (((ch & 7) ^ (i & 7)) << 4));
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint64_t x2 = pk2(__uint_as_float(w4[e] << 16), __uint_as_float(w4[e] & 0xffff0000u));
        s2 = fma2(x2, x2, s2);
      }
    }
    float a0, a1;
    upk2(s2, a0, a1);
    const float s = a0 + a1;
    sq[i] = s;
    inv_norm[i] = s > 0.f ? 1.0f / sqrtf(s) : 0.f;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async bytes -> the tensor core's view
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const float p = c.red_p;
  const int q = warp & 3, chalf = warp >> 2;
  const int halves = (b + 127) / 128;
  int nmma = 0;                                     // MMAs committed (mbarrier parity)
  for (int m = 0; m < halves; ++m) {
    const int i = m * 128 + q * 32 + lane;          // this thread's row
    const int dlo = m * 128 + q * 32;               // the warp's rows [dlo, dlo + 32)
    const bool rows_ok = dlo < b;                   // warp-uniform: the quarter holds rows < b
    const float ni = (rows_ok && i < b) ? inv_norm[i] : 0.f;
    // x_ij = g_ij / |k_j|: the row's cosine sum is ni (sum_j x_ij - x_ii), x_ii = |k_i|^2 ni;
    // cos_ij > p <=> ni x_ij > p
    uint64_t acc2[2] = {0ull, 0ull};
    int zj = -1;
    float zval = 0.f;
    for (int nh = 0; nh * 128 < b; ++nh, ++nmma) {
      const int N = min(128, b - nh * 128);         // a multiple of 16
      if (warp == 0) {
#pragma unroll
        for (int kk = 0; kk < C::KSTEPS; ++kk) {
          const uint32_t koff = (uint32_t)(kk >> 2) * slab_bytes + (uint32_t)(kk & 3) * 32u;
          umma_elect(tmem, sw128_desc(base + koff + (uint32_t)m * 128u * 128u),
                     sw128_desc(base + koff + (uint32_t)nh * 128u * 128u), idesc_bf16(128, N), kk > 0);
        }
        umma_commit_elect(smem_u32(bar));
      }
      if (warp == 0) mbar_wait_lean(smem_u32(bar), (uint32_t)(nmma & 1));   // one poller, as above
      __syncthreads();
      tc_fence_after();
      if (rows_ok) {
        const int ncw = N / 2;                      // this warp's columns: a multiple of 8
        const int tc0 = chalf * ncw;                // TMEM column of the first one
        const int jc0 = nh * 128 + tc0;             // its block column
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
        float rmx = -INFINITY;
        auto chunk8 = [&](const float* g, int jc, bool diag) {
          const float4 na = *reinterpret_cast<const float4*>(inv_norm + jc);
          const float4 nb = *reinterpret_cast<const float4*>(inv_norm + jc + 4);
          float x[8];
          const uint64_t z2 = 0ull;
          upk2(fma2(pk2(g[0], g[1]), pk2(na.x, na.y), z2), x[0], x[1]);
          upk2(fma2(pk2(g[2], g[3]), pk2(na.z, na.w), z2), x[2], x[3]);
          upk2(fma2(pk2(g[4], g[5]), pk2(nb.x, nb.y), z2), x[4], x[5]);
          upk2(fma2(pk2(g[6], g[7]), pk2(nb.z, nb.w), z2), x[6], x[7]);
          acc2[0] = add2(acc2[0], add2(pk2(x[0], x[1]), pk2(x[2], x[3])));
          acc2[1] = add2(acc2[1], add2(pk2(x[4], x[5]), pk2(x[6], x[7])));
          if (diag) {                               // warp-uniform: a lane's diagonal may be in this chunk
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = (jc + e == i) ? -INFINITY : x[e];
          }
          rmx = fmaxf(rmx, fmaxf(max3f(x[0], x[1], x[2]), max3f(x[3], x[4], max3f(x[5], x[6], x[7]))));
        };
        int c0 = 0;
        for (; c0 + 32 <= ncw; c0 += 32) {
          float g[32];
          TMEM_LD16(trow + (uint32_t)(tc0 + c0), g, 0);
          TMEM_LD16(trow + (uint32_t)(tc0 + c0 + 16), g, 16);
          tmem_wait_ld();
          // 32-column groups are 32-aligned (jc0 is), like the warp's diagonal range [dlo, dlo + 32)
          if (jc0 + c0 == dlo) {
#pragma unroll
            for (int k = 0; k < 4; ++k) chunk8(g + 8 * k, jc0 + c0 + 8 * k, true);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) chunk8(g + 8 * k, jc0 + c0 + 8 * k, false);
          }
        }
        for (; c0 < ncw; c0 += 8) {
          float g[8];
          TMEM_LD8(trow + (uint32_t)(tc0 + c0), g, 0);
          tmem_wait_ld();
          chunk8(g, jc0 + c0, jc0 + c0 + 8 > dlo && jc0 + c0 < dlo + 32);
        }
        // rare (warp-uniform): some lane has an off-diagonal cosine above p among these columns; rescan them
        // in ascending order so the last one wins
        if (__any_sync(0xffffffffu, rmx * ni > p)) {
          for (int cc = 0; cc < ncw; cc += 8) {
            float g[8];
            TMEM_LD8(trow + (uint32_t)(tc0 + cc), g, 0);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int j = jc0 + cc + e;
              const float cs = g[e] * inv_norm[j] * ni;
              if (j != i && cs > p) { zj = j; zval = cs; }
            }
          }
          if (lane == 0) *zflag = 1;
        }
      }
      tc_fence_before();
      __syncthreads();                              // TMEM reads done before the next MMA overwrites it
      tc_fence_after();
    }
    if (rows_ok && i < b) {
      float a0, a1, a2, a3;
      upk2(acc2[0], a0, a1);
      upk2(acc2[1], a2, a3);
      // the diagonal term x_ii joined the column half holding column i
      const int ncw_i = min(128, b - (i & ~127)) >> 1;  // column split of the MMA holding column i
      const float xd = (((i & 127) >= ncw_i) == (chalf == 1)) ? sq[i] * ni : 0.f;
      rsum[chalf * 256 + i] = ni * (((a0 + a1) + (a2 + a3)) - xd);
      zpart[chalf * 256 + i] = zj;
      zvpart[chalf * 256 + i] = zval;
    }
  }
  __syncthreads();
  float* out = c.ws.redund + (size_t)unit * c.max_seq_len;
  const float inv_T = 1.0f / (float)T;
  if (*zflag == 0) {                                // the common case: no cosine above p in the block
    for (int i = tid; i < nvalid; i += kRThreads) out[j0 + i] = (rsum[i] + rsum[256 + i]) * inv_T;
  } else {
  // per column i: row i's last column above p (the larger column index of the two column-split warps)
  for (int i = tid; i < b; i += kRThreads) {
    const bool up = zpart[256 + i] > zpart[i];
    zc[i] = up ? zpart[256 + i] : zpart[i];
    zv[i] = up ? zvpart[256 + i] : zvpart[i];
  }
  __syncthreads();
  // remove each column's zeroed entry from its row, in ascending column order; r[t] = sum / T
  for (int i0 = warp * 32; i0 < b; i0 += kRThreads) {
    const int i = i0 + lane;
    float s = i < b ? rsum[i] + rsum[256 + i] : 0.f;
    for (int jc = 0; jc < b; jc += 32) {
      const int key = jc + lane < b ? zc[jc + lane] : -1;
      uint32_t any = __ballot_sync(0xffffffffu, key >= 0);
      while (any) {
        const int src = __ffs(any) - 1;
        any &= any - 1;
        const int row = __shfl_sync(0xffffffffu, key, src);
        const float val = zv[jc + src];
        if (row == i) s -= val;
      }
    }
    if (i < nvalid) out[j0 + i] = s * inv_T;
  }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

template <int D>
cudaError_t launch_t(const Call& c, cudaStream_t s) {
  const int units = c.R * c.L * c.h_kv;
  // up to 3 CTAs per SM: a third CTA's copies are in flight while it waits in tcgen05.alloc for the TMEM
  // columns (256 each at b = 256) one of the other two releases
  const size_t smem = red_smem_bytes(D, c.b);
  cudaError_t e = cudaFuncSetAttribute(k_red_umma<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid(units, (c.max_seq_len + c.b - 1) / c.b);
  // K as [rows = L*N_total*b][h_kv][d]; one box = a block's b slots x 64 elements of one head (SW128)
  CUtensorMap tk;
  memset(&tk, 0, sizeof(tk));
  int ktma = 0;
  if (EncodeTiledFn enc = encode_fn()) {
    const cuuint32_t estr[3] = {1, 1, 1};
    const cuuint64_t kdim[3] = {(cuuint64_t)D, (cuuint64_t)c.h_kv, (cuuint64_t)c.L * c.N_total * c.b};
    const cuuint64_t kstr[2] = {(cuuint64_t)D * 2, (cuuint64_t)c.h_kv * D * 2};
    const cuuint32_t kbox[3] = {64, 1, (cuuint32_t)c.b};
    ktma = enc(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, c.k_cache, kdim, kstr, kbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
  }
  k_red_umma<D><<<grid, kRThreads, smem, s>>>(c, tk, ktma);
  return cudaGetLastError();
}

}  // namespace

// bf16, b % 16 == 0, 32 <= b <= 256, d in {64, 128}
cudaError_t launch_redundancy_tc(const Call& c, cudaStream_t s) {
  if (c.R * c.L * c.h_kv == 0) return cudaSuccess;
  return c.d == 128 ? launch_t<128>(c, s) : launch_t<64>(c, s);
}

}  // namespace zpc
