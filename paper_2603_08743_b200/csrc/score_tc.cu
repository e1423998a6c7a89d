// a1 + a2 on 5th-generation tensor cores (tcgen05 + TMEM + TMA), bf16 pools, sm_100a.
//
// What it computes (Alg. 1 + §C.2): for one unit (request r, layer l, KV head h)
//   x[c,t] = q_c . k_t / sqrt(d)   for the G*w window columns c = u*G + g and tokens t < T,
//   LSE[c] = log sum_{t <= T-w+u} exp x[c,t]                         (softmax normaliser, pass 1)
//   S[t]   = (1/w) sum_{u: t <= T-w+u} exp(max_g (x[(u,g),t] - LSE[(u,g)]))      (pass 2)
// i.e. softmax over each window row, max over the GQA group, mean over the window; exp is
// monotone so the max is taken before the exponential (w exps per token instead of G*w).
//
// Design (DESIGN.md §Score kernel):
//  * K is read through the block table by TMA: a 128-token tile = 128/b paged boxes of b rows x
//    64 d-elements (128B swizzle), landing in the canonical K-major SW128 UMMA layout.
//  * Pass 1 puts the window columns on M (A = Q, B = K tile): TMEM lane = column, so each epilogue
//    thread owns one column and keeps an online (max, sum) over tokens with no cross-lane work.
//  * Pass 2 flips the orientation (A = K tile, B = Q, N = G*w): TMEM lane = token, so the GQA max
//    and the window sum are in-thread over TMEM columns; S is written coalesced.
//  * A unit's tokens are split across a C-CTA cluster; partial (max, sum) per column are combined
//    through DSMEM, so pass 2 re-reads a CTA-sized slice of K (L2-resident) instead of the unit.
//  * Warp roles: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer (one thread), warps 2..9
//    epilogue (two per TMEM lane quarter). K ring of kStages smem stages, two TMEM accumulators.
#include <cuda.h>

#include <cstdlib>

#include "internal.h"

namespace zpc {
namespace {

constexpr int kTile = 128;       // tokens per tile (UMMA M in pass 2, N in pass 1)
constexpr int kStages = 4;       // K smem ring depth
constexpr int kThreads = 320;    // 10 warps
constexpr int kEpiWarps = 8;
constexpr uint32_t kTmemCols = 512;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kPolyEvery = 0;   // every k-th pass-1 exp on the FMA pipe (0 = MUFU only)

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  long long spins = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (++spins > (1LL << 26)) __trap();   // a pipeline bug must fail loudly, never hang the GPU
  }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 2^x for x <= 0 on the FMA pipe (Cody-Waite split + degree-5 minimax, rel err ~2e-7): used for a
// fraction of pass-1 exponentials so the MUFU pipe is not the only exp2 engine.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;                 // 1.5 * 2^23: round-to-nearest integer in the low bits
  const float n = t - 12582912.f;
  const float f = x - n;                          // f in [-0.5, 0.5]
  float p = 1.3534167e-4f;
  p = fmaf(p, f, 1.3395720e-3f);
  p = fmaf(p, f, 9.6180239e-3f);
  p = fmaf(p, f, 5.5504109e-2f);
  p = fmaf(p, f, 2.4022652e-1f);
  p = fmaf(p, f, 6.9314718e-1f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart (SBO).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                      // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;            // SBO
  d |= (uint64_t)1 << 46;                      // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                      // SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: bf16 x bf16 -> fp32, both operands K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
#define TMEM_LD16(taddr, v, off)                                                                          \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}," \
               " [%16];"                                                                                  \
               : "=f"(v[off + 0]), "=f"(v[off + 1]), "=f"(v[off + 2]), "=f"(v[off + 3]), "=f"(v[off + 4]),  \
                 "=f"(v[off + 5]), "=f"(v[off + 6]), "=f"(v[off + 7]), "=f"(v[off + 8]), "=f"(v[off + 9]),  \
                 "=f"(v[off + 10]), "=f"(v[off + 11]), "=f"(v[off + 12]), "=f"(v[off + 13]),              \
                 "=f"(v[off + 14]), "=f"(v[off + 15])                                                     \
               : "r"(taddr))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ float ld_dsmem_f32(const float* local, uint32_t rank) {
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
  return v;
}

// ------------------------------------------------------------------ kernel
template <int G, int W, int D, int C>
struct Cfg {
  static constexpr int GW = G * W;
  static constexpr int M1H = (GW + 127) / 128;        // pass-1 M halves (A = Q rows)
  static constexpr int NQ = M1H * 128;                 // padded Q rows in smem
  static constexpr int SLABS = D / 64;                 // 64-element (128 B) K-chunks
  static constexpr int KSTEPS = D / 16;                // UMMA K = 16 per instruction
  static constexpr int HC = (W / 2) * G;               // pass-2 columns per epilogue half
  static constexpr uint32_t Q_BYTES = NQ * D * 2;
  static constexpr uint32_t SLAB_Q = NQ * 128;         // bytes per Q slab
  static constexpr uint32_t SLAB_K = kTile * 128;      // bytes per K slab
  static constexpr uint32_t STAGE_BYTES = kTile * D * 2;
  static constexpr uint32_t OFF_K = Q_BYTES;
  static constexpr uint32_t OFF_F = OFF_K + kStages * STAGE_BYTES;   // floats: negL, pm, ps, comb
  static constexpr uint32_t OFF_BAR = OFF_F + (256 * 3 + 256) * 4;
  static constexpr uint32_t SMEM = OFF_BAR + 16 * 8 + 16 + 1024;      // + alignment slack
  static_assert(GW % 16 == 0 && GW <= 256, "pass-2 UMMA N must be a multiple of 16, <= 256");
  static_assert(HC % 16 == 0, "epilogue loads 16 columns at a time");
  static_assert(W % 2 == 0, "window split across two epilogue halves");
};

template <int G, int W, int D, int C>
__global__ void __launch_bounds__(kThreads, 1) k_score_tc(Call c, const __grid_constant__ CUtensorMap tmap_k) {
  using K = Cfg<G, W, D, C>;
  if (*c.status != ZPC_OK) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Qs = smem;
  uint8_t* Ks = smem + K::OFF_K;
  float* negL = reinterpret_cast<float*>(smem + K::OFF_F);
  float* pm = negL + 256;
  float* ps = pm + 256;
  float* comb = ps + 256;                               // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + K::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages);
  const uint32_t accf0 = smem_u32(bars + 2 * kStages), acce0 = smem_u32(bars + 2 * kStages + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x / C;
  const int rank = C > 1 ? (int)(blockIdx.x % C) : 0;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int T = c.seq_lens[r];
  const int slot = c.q_slots[r];
  const int ntot = (T + kTile - 1) / kTile;
  const int tb = (int)((long long)ntot * rank / C), te = (int)((long long)ntot * (rank + 1) / C);
  const int nt = te - tb;
  const int* table = c.tables + (size_t)r * c.table_stride;
  const int Nblk = (T + c.b - 1) / c.b;

  // ---- setup: barriers, TMEM, Q tile (swizzled by hand; zero padding rows)
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(full0 + 8 * s, 1); mbar_init(empty0 + 8 * s, 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(accf0 + 8 * a, 1); mbar_init(acce0 + 8 * a, kEpiWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_k)));
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  {
    const uint16_t* Q = reinterpret_cast<const uint16_t*>(c.q_cache);
    constexpr int CH = D / 8;                          // 16-byte chunks per row
    for (int e = threadIdx.x; e < K::NQ * CH; e += kThreads) {
      const int row = e / CH, j = e % CH;
      int4 v = make_int4(0, 0, 0, 0);
      if (row < K::GW) {
        const int u = row / G, g = row % G;
        v = *reinterpret_cast<const int4*>(Q + q_row(c, l, slot, u, h * G + g) + j * 8);
      }
      const int slab = j >> 3, jj = j & 7;
      *reinterpret_cast<int4*>(Qs + slab * K::SLAB_Q + row * 128 + ((jj ^ (row & 7)) << 4)) = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const float scale = kLog2e * rsqrtf((float)D);

  if (warp == 0) {
    // ================= TMA producer
    if (C > 1) cluster_arrive_relaxed();
    if (lane == 0) {
      const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
      const int rows_box = c.b >= kTile ? kTile : c.b;
      const int boxes = c.b >= kTile ? 1 : kTile / c.b;
      for (int i = 0; i < 2 * nt; ++i) {
        const int s = i % kStages;
        mbar_wait(empty0 + 8 * s, ((i / kStages) & 1) ^ 1);
        const int t0 = (tb + i % nt) * kTile;
        const int j0 = t0 / c.b;
        int nbox = 1;
        if (boxes > 1) nbox = min(boxes, Nblk - j0);
        mbar_expect_tx(full0 + 8 * s, (uint32_t)(nbox * rows_box * 128 * K::SLABS));
        const uint32_t dst = smem_u32(Ks + s * K::STAGE_BYTES);
        for (int bx = 0; bx < nbox; ++bx) {
          const int blk = table[j0 + bx];
          const int row = (int)(((long long)l * c.N_total + blk) * c.b + (boxes > 1 ? 0 : t0 % c.b));
          for (int sl = 0; sl < K::SLABS; ++sl)
            tma_load_3d(dst + sl * K::SLAB_K + bx * rows_box * 128, &tmap_k, sl * 64, h, row, full0 + 8 * s,
                        i < nt ? keep : drop);
        }
      }
    }
    __syncwarp();
    if (C > 1) cluster_wait();
  } else if (warp == 1) {
    // ================= MMA issuer (single thread)
    if (C > 1) cluster_arrive_relaxed();
    if (lane == 0) {
      const uint32_t qb = smem_u32(Qs);
      for (int i = 0; i < 2 * nt; ++i) {
        const int s = i % kStages, a = i & 1;
        mbar_wait(acce0 + 8 * a, ((i >> 1) & 1) ^ 1);
        mbar_wait(full0 + 8 * s, (i / kStages) & 1);
        tc_fence_after();
        const uint32_t kb = smem_u32(Ks + s * K::STAGE_BYTES);
        const uint32_t dacc = tmem + a * 256;
        if (i < nt) {
#pragma unroll
          for (int half = 0; half < K::M1H; ++half)
#pragma unroll
            for (int k = 0; k < K::KSTEPS; ++k) {
              const uint64_t ad = sw128_desc(qb + (k >> 2) * K::SLAB_Q + half * 128 * 128 + (k & 3) * 32);
              const uint64_t bd = sw128_desc(kb + (k >> 2) * K::SLAB_K + (k & 3) * 32);
              umma(dacc + half * 128, ad, bd, idesc_bf16(128, kTile), k > 0);
            }
        } else {
#pragma unroll
          for (int k = 0; k < K::KSTEPS; ++k) {
            const uint64_t ad = sw128_desc(kb + (k >> 2) * K::SLAB_K + (k & 3) * 32);
            const uint64_t bd = sw128_desc(qb + (k >> 2) * K::SLAB_Q + (k & 3) * 32);
            umma(dacc, ad, bd, idesc_bf16(kTile, K::GW), k > 0);
          }
        }
        umma_commit(empty0 + 8 * s);
        umma_commit(accf0 + 8 * a);
      }
    }
    __syncwarp();
    if (C > 1) cluster_wait();
  } else {
    // ================= epilogue warps
    const int ew = warp - 2;
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = ew >> 2;
    const int col = half * 128 + q * 32 + lane;
    const bool warp_cols = (half * 128 + q * 32) < K::GW;
    const bool col_ok = col < K::GW;
    const int u1 = col_ok ? col / G : 0;
    const int limit1 = T - W + u1;          // pass-1 causal limit of this column (R1, R2)
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    float m = -INFINITY, ssum = 0.f;
    for (int i = 0; i < 2 * nt; ++i) {
      const int a = i & 1;
      mbar_wait(accf0 + 8 * a, (i >> 1) & 1);
      tc_fence_after();
      const int t0 = (tb + i % nt) * kTile;
      if (i < nt) {
        // ---- pass 1: this thread owns window column `col`; 128 token logits in TMEM columns,
        //      consumed as two 64-column batches with an online (max, sum) update.
#pragma unroll 1
        for (int bh = 0; bh < 2; ++bh) {
          float v[64];
          if (warp_cols) {
#pragma unroll
            for (int k = 0; k < 4; ++k) TMEM_LD16(lane_base + a * 256 + half * 128 + bh * 64 + k * 16, v, k * 16);
            tmem_wait_ld();
          }
          if (bh == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acce0 + 8 * a);
          }
          if (col_ok) {
            const int tbase = t0 + bh * 64;
            if (tbase + 63 > limit1) {
#pragma unroll
              for (int j = 0; j < 64; ++j)
                if (tbase + j > limit1) v[j] = -INFINITY;
            }
            float mp[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) mp[j] = v[j];
#pragma unroll
            for (int j = 8; j < 64; ++j) mp[j & 7] = fmaxf(mp[j & 7], v[j]);
            const float mx = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                                   fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
            if (mx > -INFINITY) {
              const float mn = fmaxf(m, mx * scale);
              float sp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
              for (int j = 0; j < 64; ++j) {
                const float arg = fmaf(v[j], scale, -mn);
                sp[j & 3] += (kPolyEvery > 0 && (j % kPolyEvery) == kPolyEvery - 1) ? ex2_poly(arg) : ex2f(arg);
              }
              ssum = (m > -INFINITY ? ssum * ex2f(m - mn) : 0.f) + ((sp[0] + sp[1]) + (sp[2] + sp[3]));
              m = mn;
            }
          }
        }
      } else {
        // ---- pass 2: this thread owns token t0 + q*32 + lane and the window rows of its half;
        //      columns stream in batches of <= 64; (u, g) of every column is a compile-time constant.
        const int t = t0 + q * 32 + lane;
        const int du = t - (T - W) - half * (W / 2);   // window row uu of this half is causal iff uu >= du
        const float4* nl4 = reinterpret_cast<const float4*>(negL + half * K::HC);
        float acc0 = 0.f, acc1 = 0.f, mx = 0.f;
        constexpr int NCH = K::HC / 16;
#pragma unroll
        for (int b0 = 0; b0 < NCH; b0 += 4) {
          float v[64];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (b0 + k < NCH) TMEM_LD16(lane_base + a * 256 + half * K::HC + (b0 + k) * 16, v, k * 16);
          tmem_wait_ld();
          if (b0 + 4 >= NCH) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acce0 + 8 * a);
          }
#pragma unroll
          for (int j4 = 0; j4 < 16; ++j4) {
            if (b0 * 16 + j4 * 4 < K::HC) {
              const float4 L4 = nl4[b0 * 4 + j4];
              const float Lv[4] = {L4.x, L4.y, L4.z, L4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int cc = b0 * 16 + j4 * 4 + e;      // column within the half (compile time)
                const int uu = cc / G, g = cc % G;
                const float y = fmaf(v[j4 * 4 + e], scale, Lv[e]);
                mx = (g == 0) ? y : fmaxf(mx, y);
                if (g == G - 1) {
                  const float pterm = (uu >= du) ? ex2f(mx) : 0.f;
                  if (uu & 1) acc1 += pterm; else acc0 += pterm;
                }
              }
            }
          }
        }
        const float acc = acc0 + acc1;
        float* cb = comb + (i & 1) * kTile;
        if (half == 1) cb[q * 32 + lane] = acc;
        named_bar(1, kEpiWarps * 32);
        if (half == 0 && t < T)
          c.ws.scores[(size_t)unit * c.max_seq_len + t] = (acc + cb[q * 32 + lane]) * (1.0f / W);
      }
      if (i == nt - 1) {
        // ---- end of pass 1: LSE per column (combined across the cluster through DSMEM)
        if (C == 1) {
          if (col_ok) {
            const float L2 = m + lg2f(ssum);
            negL[col] = -L2;
            c.ws.lse[(size_t)unit * K::GW + col] = L2;
          }
        } else {
          if (col_ok) { pm[col] = m; ps[col] = ssum; }
          cluster_arrive_release();
          cluster_wait();
          if (col_ok) {
            float M = -INFINITY;
#pragma unroll
            for (int rr = 0; rr < C; ++rr) M = fmaxf(M, ld_dsmem_f32(pm + col, rr));
            float S = 0.f;
#pragma unroll
            for (int rr = 0; rr < C; ++rr) {
              const float mr = ld_dsmem_f32(pm + col, rr);
              if (mr > -INFINITY) S += ld_dsmem_f32(ps + col, rr) * ex2f(mr - M);
            }
            const float L2 = M + lg2f(S);
            negL[col] = -L2;
            if (rank == 0) c.ws.lse[(size_t)unit * K::GW + col] = L2;
          }
        }
        named_bar(1, kEpiWarps * 32);
      }
    }
    if (nt == 0 && C > 1) {
      // this CTA got no tiles: publish an empty partial and take part in the exchange
      if (col_ok) { pm[col] = -INFINITY; ps[col] = 0.f; }
      cluster_arrive_release();
      cluster_wait();
    }
  }
  // ---- teardown
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  if (C > 1) {
    cluster_arrive_release();   // no CTA leaves while a peer may still read its pm/ps
    cluster_wait();
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;   // resolved driver entry point (process-wide, immutable)
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

template <int G, int W, int D, int C>
cudaError_t launch_tc(const Call& c, const CUtensorMap& tm, cudaStream_t s) {
  using K = Cfg<G, W, D, C>;
  auto kern = k_score_tc<G, W, D, C>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
  if (e != cudaSuccess) return e;
  const int units = c.R * c.L * c.h_kv;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * C);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, c, tm);
}

// Cluster size: CTAs per unit. Splitting a unit's tokens over C CTAs shrinks the K slice each
// CTA re-reads in pass 2 (in flight across the GPU: ~148/C slices), keeping it L2-resident
// (DESIGN.md §Score kernel, L2 reuse). ZPC_SCORE_CLUSTER (1/2/4) overrides, for tuning runs.
int cluster_size(const Call& c) {
  if (const char* e = getenv("ZPC_SCORE_CLUSTER")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4) return v;
  }
  if (c.max_seq_len < 2 * kTile) return 1;
  if (c.max_seq_len < 16 * kTile) return 2;
  return 4;
}

template <int G, int W, int D>
cudaError_t launch_c(const Call& c, const CUtensorMap& tm, cudaStream_t s) {
  switch (cluster_size(c)) {
    case 4: return launch_tc<G, W, D, 4>(c, tm, s);
    case 2: return launch_tc<G, W, D, 2>(c, tm, s);
    default: return launch_tc<G, W, D, 1>(c, tm, s);
  }
}

template <int D>
cudaError_t dispatch_g(const Call& c, const CUtensorMap& tm, cudaStream_t s, bool* used) {
  if (c.w != 32) return cudaSuccess;
  *used = true;
  switch (c.G) {
    case 4: return launch_c<4, 32, D>(c, tm, s);
    case 5: return launch_c<5, 32, D>(c, tm, s);
    case 7: return launch_c<7, 32, D>(c, tm, s);
    case 8: return launch_c<8, 32, D>(c, tm, s);
    default: *used = false; return cudaSuccess;
  }
}

}  // namespace

cudaError_t launch_score_tc(const Call& c, cudaStream_t s, bool* used) {
  *used = false;
  if (c.dtype != ZPC_BF16) return cudaSuccess;
  const bool b_ok = (c.b >= 8 && kTile % c.b == 0) || (c.b % kTile == 0);
  if (!b_ok || (c.d != 64 && c.d != 128)) return cudaSuccess;
  if (c.R * c.L * c.h_kv == 0) { *used = true; return cudaSuccess; }
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaSuccess;
  CUtensorMap tm;
  const cuuint64_t gdim[3] = {(cuuint64_t)c.d, (cuuint64_t)c.h_kv, (cuuint64_t)c.L * c.N_total * c.b};
  const cuuint64_t gstride[2] = {(cuuint64_t)c.d * 2, (cuuint64_t)c.h_kv * c.d * 2};
  const cuuint32_t box[3] = {64, 1, (cuuint32_t)(c.b >= kTile ? kTile : c.b)};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, c.k_cache, gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaSuccess;   // not expressible as a tensor map: CUDA-core path
  return c.d == 64 ? dispatch_g<64>(c, tm, s, used) : dispatch_g<128>(c, tm, s, used);
}

}  // namespace zpc
