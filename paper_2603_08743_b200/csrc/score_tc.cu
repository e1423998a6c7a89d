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
//    epilogue (two per TMEM lane quarter). K ring of K::ST smem stages, two TMEM accumulators,
//    persistent CTAs looping over units, Q double-buffered by TMA.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include <cuda_bf16.h>
#include <type_traits>

#include "internal.h"
#include "tc_util.h"

namespace zpc {
namespace {

constexpr int kThreads = 512;    // 16 warps: Q-TMA, MMA, (idle), feeder, 4 K loaders, 8 epilogue
constexpr int kLoadWarps = 4;
constexpr int kEpiWarp0 = 8;     // first epilogue warp (warps 8..15: lane quarter = warp % 4)
#ifndef ZPC_POLY
#define ZPC_POLY 0
#endif
// ZPC_POLY = k: k of every 8 pass-1 exp2 pairs on the FMA pipe (ex2_poly2) instead of MUFU.
// ZPC_POLY_SPLIT: the same for k_score_ovl's token-split instances (G*w <= 128), where the two warps
// of a lane quarter both run the pass-1 exp chain and the MUFU is the busiest pipe. Measured on one
// B200 (gpurun_out A/B, score ms): llama8b (G*w = 128) 13.13 / 12.36 / 12.46 / 13.02 / 13.40 for
// k = 0 / 1 / 2 / 3 / 4; qwen7b (G*w = 224) 8.07 / 8.17 / 8.46 / 8.71 / 9.03 -> defaults 0 and 1.
#ifndef ZPC_POLY_SPLIT
#define ZPC_POLY_SPLIT 1
#endif
#ifndef ZPC_POLY_TC   // k_score_tc's pass 1 (the w = 16 calls of the paper's operating point)
#define ZPC_POLY_TC ZPC_POLY
#endif
constexpr int kPolyEighths = ZPC_POLY;
__host__ __device__ constexpr bool poly_pair(int j, int pe = kPolyEighths) { return pe != 0 && (j & 7) >= 8 - pe; }
constexpr int kEpiWarps = 8;
// setmaxnreg budget: 8 producer warps x kProdRegs + 8 epilogue warps x kEpiRegs <= 64K registers
constexpr int kProdRegs = 72;
constexpr int kEpiRegs = 184;
static_assert(8 * kProdRegs + 8 * kEpiRegs <= 2048, "register file: 65536 = 32 lanes x 2048");
constexpr uint32_t kL1Reserve = 0;   // L1 left unallocated (cp.async does not need it: measured)


// ------------------------------------------------------------------ kernel
template <int G, int W, int D, int C>
struct Cfg {
  static constexpr int GW = G * W;
  static constexpr int M1H = (GW + 127) / 128;        // pass-1 M halves (A = Q rows; rows >= GW are
                                                      // whatever follows in smem: their D rows are unused)
  static constexpr int SLABS = D / 64;                 // 64-element (128 B) K-chunks
  static constexpr int KSTEPS = D / 16;                // UMMA K = 16 per instruction
  static constexpr int HC = (W / 2) * G;               // pass-2 columns per epilogue half
  static constexpr int UB = 4;                         // window rows per pass-2 batch
  static constexpr int LDMAX = (UB * G + 15) / 16 + 1;  // 16-column TMEM loads per batch (upper bound)
  static constexpr uint32_t SLAB_Q = GW * 128;         // bytes per Q slab (GW rows of 128 B)
  static constexpr uint32_t Q_BYTES = SLAB_Q * SLABS;
  static constexpr uint32_t SLAB_K = kTile * 128;      // bytes per K slab
  static constexpr uint32_t STAGE_BYTES = kTile * D * 2;
  static constexpr uint32_t MISC = (2 * 256 * 2 + 256 + 2 * kTile) * 4 + kIdSlots * kMaxIds * 4 + 56 * 8 + 16;
  // Shared memory and L1 are one 228 KB array on sm_100: the cp.async gather stages its in-flight
  // lines through L1, so the kernel leaves kL1Reserve bytes of it unallocated (DESIGN.md §Score
  // kernel, "L1 is the gather's in-flight buffer"). Q is therefore single-buffered.
  // pass-2 normaliser folded into the MMA (a 9th K-step, no-swizzle K-major core matrices of
  // 8 rows x 16 B; LBO = 128 B between the two K halves, SBO = 256 B between 8-row groups):
  //   A_aug [kTile x 16] = ones in k = 0..2,  B_aug [GW x 16] = bf16 split (hi, mid, lo) of -L2/s
  // so the pass-2 accumulator holds q.k - L2/s directly.
  static constexpr uint32_t AUG_A_BYTES = kTile * 32;
  static constexpr uint32_t AUG_B_BYTES = GW * 32;
  static constexpr uint32_t OFF_AUG_A = Q_BYTES;
  static constexpr uint32_t OFF_AUG_B = OFF_AUG_A + AUG_A_BYTES;
  static constexpr uint32_t AUG_END = (OFF_AUG_B + AUG_B_BYTES + 1023) / 1024 * 1024;
  static constexpr int STAGES_FIT = (int)((227 * 1024 - kL1Reserve - 1024 - MISC - AUG_END) / STAGE_BYTES);
  static constexpr int ST = STAGES_FIT > 6 ? 6 : STAGES_FIT;   // K ring depth
  static constexpr uint32_t OFF_Q0 = 0;
  static constexpr uint32_t OFF_K = AUG_END;
  static constexpr uint32_t OFF_F = OFF_K + ST * STAGE_BYTES;        // floats
  static constexpr uint32_t OFF_IDS = OFF_F + (2 * 256 * 2 + 256 + 2 * kTile) * 4;
  static constexpr uint32_t OFF_BAR = OFF_IDS + kIdSlots * kMaxIds * 4;
  static constexpr uint32_t SMEM = OFF_BAR + 56 * 8 + 16 + 1024;     // + alignment slack
  static_assert(GW % 16 == 0 && GW <= 256, "pass-2 UMMA N must be a multiple of 16, <= 256");
  static_assert(W == 32 || W == 16, "epilogue batching assumes w = 32 (configs) or 16 (the paper's, PAPER.md:162)");
  static_assert(ST >= 2, "K ring needs >= 2 stages");
  static_assert(Q_BYTES % 1024 == 0, "Q slabs must stay 1024-B aligned for SW128");
};

// 2^x on MUFU for most pairs, on the FMA pipe for ZPC_POLY of every 8 pairs: balances the two pipes.
template <int J>
__device__ __forceinline__ uint64_t ex2_pair(uint64_t a2) {
  if constexpr (poly_pair(J, kPolyEighths)) {
    return ex2_poly2(a2);
  } else {
    float a0, a1;
    upk2(a2, a0, a1);
    return pk2(ex2f(a0), ex2f(a1));
  }
}

// sum_j 2^(v[j]*scale - m) over a 64-value batch, packed
template <int J>
__device__ __forceinline__ void sum_exp_rec(const float* v, uint64_t S2, uint64_t NM2, uint64_t* acc) {
  if constexpr (J < 32) {
    const uint64_t arg = fma2(pk2(v[2 * J], v[2 * J + 1]), S2, NM2);
    acc[J & 3] = add2(acc[J & 3], ex2_pair<J>(arg));
    sum_exp_rec<J + 1>(v, S2, NM2, acc);
  }
}
template <int N, int PE = kPolyEighths>
__device__ __forceinline__ float sum_exp_n(const float* v, float scale, float m) {
  uint64_t acc[4] = {0, 0, 0, 0};
  const uint64_t S2 = pk2(scale, scale), NM2 = pk2(-m, -m);
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const uint64_t arg = fma2(pk2(v[2 * j], v[2 * j + 1]), S2, NM2);
    if (poly_pair(j, PE)) {
      acc[j & 3] = add2(acc[j & 3], ex2_poly2(arg));
    } else {
      float a0, a1;
      upk2(arg, a0, a1);
      acc[j & 3] = add2(acc[j & 3], pk2(ex2f(a0), ex2f(a1)));
    }
  }
  const uint64_t s2 = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
  float a, b;
  upk2(s2, a, b);
  return a + b;
}
__device__ __forceinline__ float sum_exp64(const float* v, float scale, float m) {
  uint64_t acc[4] = {0, 0, 0, 0};
  sum_exp_rec<0>(v, pk2(scale, scale), pk2(-m, -m), acc);
  const uint64_t s2 = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
  float a, b;
  upk2(s2, a, b);
  return a + b;
}

template <int G, int W, int D, int C>
__global__ void __launch_bounds__(kThreads, 1) k_score_tc(Call c, const __grid_constant__ CUtensorMap tmap_q) {
  using K = Cfg<G, W, D, C>;
  if (*c.status != ZPC_OK) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Ks = smem + K::OFF_K;
  float* pmv = reinterpret_cast<float*>(smem + K::OFF_F);   // [2][256] partial max (by unit parity)
  float* psv = pmv + 512;                                     // [2][256] partial sums
  float* negL = psv + 512;                                    // [256]
  float* comb = negL + 256;                                   // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + K::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 54);
  int* ids = reinterpret_cast<int*>(smem + K::OFF_IDS);                  // [kIdSlots][kMaxIds]
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + 40);
  const uint32_t accf0 = smem_u32(bars + 8), acce0 = smem_u32(bars + 10);
  const uint32_t qfull0 = smem_u32(bars + 12), qempty0 = smem_u32(bars + 14);
  const uint32_t xchg0 = smem_u32(bars + 16);
  const uint32_t augf = smem_u32(bars + 18);                  // B_aug of the current unit written

  // warp index broadcast from lane 0: the compiler then treats it (and what it guards) as warp-uniform
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int rank = C > 1 ? (int)(blockIdx.x % C) : 0;
  const int cluster_id = blockIdx.x / C;
  const int nclusters = gridDim.x / C;
  const int units = c.R * c.L * c.h_kv;

  if (threadIdx.x == 0) {
    for (int s = 0; s < K::ST; ++s) { mbar_init(full0 + 8 * s, kLoadWarps * 32); mbar_init(empty0 + 8 * s, 1); }
    for (int a = 0; a < 2; ++a) {
      mbar_init(accf0 + 8 * a, 1);
      mbar_init(acce0 + 8 * a, kEpiWarps);
      mbar_init(qfull0 + 8 * a, 1);
      mbar_init(qempty0 + 8 * a, 1);
      mbar_init(xchg0 + 8 * a, C);
    }
    mbar_init(augf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_q)));
  }
  {
    // A_aug rows: bf16 1.0 in k = 0..2, zeros elsewhere; B_aug starts all zero (k = 3..15 stay 0)
    uint4* aug = reinterpret_cast<uint4*>(smem + K::OFF_AUG_A);
    for (int i = threadIdx.x; i < (int)((K::AUG_A_BYTES + K::AUG_B_BYTES) / 16); i += kThreads) {
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      // 16-B chunk i of A_aug: (group, khalf, row%8) = (i / 16, (i / 8) & 1, i % 8); khalf 0 holds k 0..7
      if (i < (int)(K::AUG_A_BYTES / 16) && ((i >> 3) & 1) == 0) v = make_uint4(0x3F803F80u, 0x00003F80u, 0u, 0u);
      aug[i] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (C > 1) cluster_sync_all();        // peers' barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);   // warp-uniform TMEM base
  const float scale = kLog2e * rsqrtf((float)D);

  // per-unit geometry, identical in every role
  // NEXT-4 (ZPC_F_LSE_INPUT): the normalisers are an input, so a unit runs only pass 2 (p1 = 0)
  const bool one_pass = c.lse_in != nullptr;
  struct UnitInfo { int r, l, h, T, slot, tb, nt, p1, id; };
  // work index -> unit: (layer, head)-major with the requests inner for single-pass shared-prefix calls, so the
  // clusters working at the same time read the same prefix tiles (one DRAM read, the rest from L2: the prefix
  // dedup of PAPER.md:131); unit order otherwise
  const bool lh_major = one_pass && (c.flags & ZPC_F_PREFIX) && !(c.debug & 8192u);
  auto unit_info = [&](int v) {
    UnitInfo u;
    const int unit = lh_major ? (v % c.R) * (c.L * c.h_kv) + v / c.R : v;
    u.id = unit;
    u.h = unit % c.h_kv;
    u.l = (unit / c.h_kv) % c.L;
    u.r = unit / (c.h_kv * c.L);
    u.T = c.seq_lens[u.r];
    u.slot = c.q_slots[u.r];
    const int ntot = (u.T + kTile - 1) / kTile;
    u.tb = (int)((long long)ntot * rank / C);
    u.nt = (int)((long long)ntot * (rank + 1) / C) - u.tb;
    u.p1 = one_pass ? 0 : u.nt;          // pass-1 steps; the unit has p1 + nt steps in all
    return u;
  };
  // step i of a unit -> tile index: pass 1 ascending, pass 2 DESCENDING (the most recently
  // streamed tiles are the ones most likely still in L2)
  auto tile_of = [](const UnitInfo& u, int i) { return i < u.p1 ? u.tb + i : u.tb + (u.p1 + u.nt - 1 - i); };

  // register rebalance per warpgroup (setmaxnreg must dominate each role's code so ptxas
  // allocates the epilogue with kEpiRegs): the producers need few registers, the epilogue's latency
  // hiding (batches in flight, hoisted TMEM loads) needs many
  if (warp < kEpiWarp0) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs));
  if (warp == 0) {
    // ================= Q producer: one TMA box per 64-element slab per unit (double buffer)
    if (lane == 0) {
      const uint64_t drop = policy_evict_first();
      for (int it = 0, unit = cluster_id; unit < units; ++it, unit += nclusters) {
        const UnitInfo u = unit_info(unit);
        const int qb = 0;                    // single Q buffer (see kL1Reserve)
        mbar_wait_backoff(qempty0, (it & 1) ^ 1, 2000);
        if (c.debug & 32u) { mbar_arrive(qfull0); continue; }   // bisection: no Q load
        mbar_expect_tx(qfull0, K::Q_BYTES);
        const uint32_t qdst = smem_u32(smem + K::OFF_Q0);
        const int qrow = (u.l * c.M + u.slot) * W;
        for (int sl = 0; sl < K::SLABS; ++sl)
          tma_load_3d(qdst + sl * K::SLAB_Q, &tmap_q, sl * 64, u.h * G, qrow, qfull0 + 8 * qb, drop);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 4 + kLoadWarps && (c.debug & 2048u)) {
    // bisection: no loaders (the feeder is off too)
  } else if (warp >= 4 && warp < 4 + kLoadWarps) {
    // ---- K gather by the loader warps: rows through the block table (ids from the walker), 16-B
    // cp.async each (D/8 threads per 2*D-byte row, coalesced), written straight into the SW128
    // K-major layout; the stage's mbarrier counts every thread once its copies land. Step k+ST
    // is issued right after acc_full(k) proved MMA(k) -- the last reader of stage k%ST -- done.
    constexpr int CPR = D / 8;                       // 16-B chunks per row
    constexpr int RPP = kLoadWarps * 32 / CPR;       // rows per pass
    static_assert(RPP % 8 == 0, "the per-thread SW128 swizzle term needs rows-per-pass % 8 == 0");
    const int et = threadIdx.x - 4 * 32;
    const int cr = et % CPR, rsub = et / CPR;
    const uint32_t chunk_off = (uint32_t)(cr >> 3) * K::SLAB_K;
    const uint16_t* Kg = reinterpret_cast<const uint16_t*>(c.k_cache);
    const uint32_t ids_base = smem_u32(ids);
    const bool b_pow2 = (c.b & (c.b - 1)) == 0;
    const int b_log2 = 31 - __clz(c.b);
    // load cursor (may run ahead into the next units); the tile's block ids come from the walker
    int ld_unit = cluster_id, ld_i = 0, ld_step = 0;
    UnitInfo ld_u = ld_unit < units ? unit_info(ld_unit) : UnitInfo{};
    // per-thread constants of the gather: rows RPP*k + rsub, 16-B chunk cr; (row & 7) == (rsub & 7)
    // because RPP is a multiple of 8, so the SW128 swizzle term is constant per thread
    const uint32_t dst_thr = (uint32_t)rsub * 128u + (uint32_t)(((cr & 7) ^ (rsub & 7)) << 4) + chunk_off;
    const uint32_t hD = (uint32_t)c.h_kv * D;              // elements between consecutive slots
    auto issue_next_load = [&]() {
      while (ld_unit < units && ld_i >= ld_u.p1 + ld_u.nt) {
        ld_unit += nclusters;
        ld_i = 0;
        if (ld_unit < units) ld_u = unit_info(ld_unit);
      }
      if (ld_unit >= units) return;
      const int st = ld_step % K::ST;
      const int t0 = tile_of(ld_u, ld_i) * kTile;
      const int j0 = b_pow2 ? (t0 >> b_log2) : t0 / c.b;
      const int T = ld_u.T;
      // 64-bit base of (layer, head, chunk); per-row offsets fit 32 bits (one layer < 2^31 elements)
      const uint16_t* lbase = Kg + (size_t)ld_u.l * c.N_total * c.b * hD + (size_t)ld_u.h * D + cr * 8;
      const uint32_t dst0 = smem_u32(Ks + st * K::STAGE_BYTES) + dst_thr;
      if ((c.debug & 1u) && blockIdx.x == 0 && lane == 0 && ld_step < 256)
        reinterpret_cast<unsigned long long*>(c.ws.kept)[4096 + ld_step * 16 + (warp - 4)] = gtimer();
      if ((c.debug & 1u) && blockIdx.x == 0 && et == 0 && ld_step < 512)
        reinterpret_cast<unsigned long long*>(c.ws.kept)[ld_step * 4 + 0] = gtimer();
      named_bar(4, kLoadWarps * 32 + 32);                     // feeder: ids of this tile, stage free
      // all block ids first (explicit ld.shared: a generic load would queue behind the copies)
      const uint32_t sid = ids_base + (uint32_t)(ld_step % kIdSlots) * kMaxIds * 4;
      if (c.b == 16 && !(c.debug & 256u)) {
        // block-major fast path (b = 16): one id per block, this thread's 16/RPP rows of the block
        // at a constant stride -- few instructions per cp.async (the gather shares its SMSPs with
        // the MUFU-bound epilogue, so its instruction count is its throughput; measured)
        constexpr int RB = 16 / RPP;                         // rows of a block per thread
        constexpr int NBLK = kTile / 16;
        const uint32_t qstride = (uint32_t)RPP * hD;
        const uint32_t rbase = (uint32_t)rsub * hD;
        int blk[NBLK];
#pragma unroll
        for (int jb = 0; jb < NBLK; ++jb) {
          blk[jb] = lds_s32(sid + 4u * (uint32_t)jb);
          ZPC_CHECK(t0 + jb * 16 >= T || (blk[jb] >= 0 && blk[jb] < c.N_total));
        }
        if (t0 + kTile <= T) {                               // full tile: no predicates
#pragma unroll
          for (int jb = 0; jb < NBLK; ++jb) {
            uint32_t off = (uint32_t)blk[jb] * 16u * hD + rbase;
#pragma unroll
            for (int q = 0; q < RB; ++q, off += qstride)
              cp_async16(dst0 + (uint32_t)((jb * 16 + q * RPP) * 128), lbase + off);
          }
        } else {
#pragma unroll
          for (int jb = 0; jb < NBLK; ++jb) {
            uint32_t off = (uint32_t)blk[jb] * 16u * hD + rbase;
#pragma unroll
            for (int q = 0; q < RB; ++q, off += qstride)
              if (t0 + jb * 16 + q * RPP + rsub < T)
                cp_async16(dst0 + (uint32_t)((jb * 16 + q * RPP) * 128), lbase + off);
          }
        }
      } else {
        uint32_t off[kTile / RPP];
#pragma unroll
        for (int k = 0; k < kTile / RPP; ++k) {
          const int t = t0 + RPP * k + rsub;
          const int jr = b_pow2 ? (t >> b_log2) : t / c.b;
          const int blk = lds_s32(sid + 4u * (uint32_t)min(max(jr - j0, 0), kMaxIds - 1));
          ZPC_CHECK(t >= T || (blk >= 0 && blk < c.N_total && t - jr * c.b < c.b));
          off[k] = ((uint32_t)blk * (uint32_t)c.b + (uint32_t)(t - jr * c.b)) * hD;
        }
        if (!(c.debug & 256u)) {
#pragma unroll
          for (int k = 0; k < kTile / RPP; ++k)
            if (t0 + RPP * k + rsub < T) cp_async16(dst0 + (uint32_t)(RPP * k * 128), lbase + off[k]);
        }
      }
      cp_async_arrive_noinc(full0 + 8 * st);
      if ((c.debug & 1u) && blockIdx.x == 0 && lane == 0 && ld_step < 256)
        reinterpret_cast<unsigned long long*>(c.ws.kept)[4096 + ld_step * 16 + 8 + (warp - 4)] = gtimer();
      ++ld_i;
      ++ld_step;
    };
    while (ld_unit < units) issue_next_load();

  } else if (warp == 3 && !(c.debug & 2048u)) {
    // ================= feeder: for every K tile, in the loaders' order, the block ids and the
    // stage's release by the MMA (the empty mbarrier, polled here only); then one named barrier
    // with the 128 gathering threads publishes both. The loaders block in bar.sync instead of
    // polling (their polls cost issue slots on SMSPs the MUFU-bound epilogue shares; measured).
    // The ids are copied table -> smem ring by 4-byte cp.async kIdAhead tiles ahead of the one
    // being published, so the table load latency is off the per-tile critical path (a load issued
    // per tile right before its publication made every tile wait one L2/DRAM round trip:
    // measured ~1500 cycles per step with the gather, MMA and epilogue all disabled).
    // Ring slot (g % kIdSlots) is rewritten at iteration g - kIdAhead, i.e. before barrier
    // g - kIdAhead; the loaders finished reading tile g - kIdSlots's slot before they reached
    // barrier g - kIdSlots + 1 <= g - kIdAhead - 1 (kIdSlots >= kIdAhead + 2).
    static_assert(kIdSlots >= kIdAhead + 2, "id ring too small for the lookahead");
    int l_unit = cluster_id, l_i = 0;            // load cursor (kIdAhead tiles ahead)
    UnitInfo l_u = l_unit < units ? unit_info(l_unit) : UnitInfo{};
    int p_unit = cluster_id, p_i = 0;            // publish cursor
    UnitInfo p_u = l_u;
    const uint32_t ids_base = smem_u32(ids);
    auto issue_ids = [&](int slot) {
      while (l_unit < units && l_i >= l_u.p1 + l_u.nt) {
        l_unit += nclusters;
        l_i = 0;
        if (l_unit < units) l_u = unit_info(l_unit);
      }
      if (l_unit < units) {
        const int t0 = tile_of(l_u, l_i) * kTile;
        const int j0 = t0 / c.b;
        const int nb = (min(t0 + kTile, l_u.T) - 1) / c.b - j0 + 1;
        if (lane < nb)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ids_base + (uint32_t)(slot * kMaxIds + lane) * 4u),
                       "l"(c.tables + (size_t)l_u.r * c.table_stride + j0 + lane) : "memory");
        ++l_i;
      }
      asm volatile("cp.async.commit_group;" ::: "memory");   // one group per tile (possibly empty)
    };
#pragma unroll 1
    for (int k = 0; k < kIdAhead; ++k) issue_ids(k);
    for (int g = 0;; ++g) {
      while (p_unit < units && p_i >= p_u.p1 + p_u.nt) {
        p_unit += nclusters;
        p_i = 0;
        if (p_unit < units) p_u = unit_info(p_unit);
      }
      if (p_unit >= units) break;
      issue_ids((g + kIdAhead) % kIdSlots);
      if (g >= K::ST) {   // stage reuse: the MMAs that read it are complete
        if (lane == 0) mbar_wait(empty0 + 8 * (g % K::ST), ((g / K::ST) & 1) ^ 1);
        __syncwarp();
      }
      asm volatile("cp.async.wait_group %0;" ::"n"(kIdAhead) : "memory");   // tile g's ids landed
      named_bar(4, kLoadWarps * 32 + 32);
      ++p_i;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == 1) {
    // ================= MMA issuer: the whole warp runs converged (descriptors are warp-uniform,
    // so ptxas keeps them in uniform registers) and one elected lane issues each tcgen05.mma /
    // commit; a lane-0-only region made ptxas wrap every MMA in an ELECT/R2UR/BRA.U.ANY loop
    // (~100 cycles per issue, measured: the 9-MMA pass-2 step could not keep the tensor pipe fed).
    // Each epilogue warp waits the commit mbarrier of its step itself.
    int kstep = 0, astep = 0;
    const uint64_t aug_a = none_desc(smem_u32(smem + K::OFF_AUG_A), 128, 256);
    const uint64_t aug_b = none_desc(smem_u32(smem + K::OFF_AUG_B), 128, 256);
    const uint64_t qd0 = sw128_desc(smem_u32(smem + K::OFF_Q0));
    for (int it = 0, unit = cluster_id; unit < units; ++it, unit += nclusters) {
      const UnitInfo uu = unit_info(unit);
      // step counts broadcast from lane 0 so the loop control (and every descriptor) stays in
      // uniform registers: no R2UR moves around each tcgen05.mma
      const int p1 = __shfl_sync(0xffffffffu, uu.p1, 0), nsteps = __shfl_sync(0xffffffffu, uu.p1 + uu.nt, 0);
      mbar_wait(qfull0, it & 1);
      for (int i = 0; i < nsteps; ++i, ++kstep, ++astep) {
        const int s = kstep % K::ST, a = astep & 1;
        const bool mrec = (c.debug & 1u) && blockIdx.x == 0 && astep < 1024 && lane == 0;
        unsigned long long* mdbg = reinterpret_cast<unsigned long long*>(c.ws.kept);
        if (mrec) mdbg[16384 + astep * 4 + 0] = gtimer();
        mbar_wait(acce0 + 8 * a, ((astep >> 1) & 1) ^ 1);
        if (mrec) mdbg[16384 + astep * 4 + 1] = gtimer();
        if (!(c.debug & 2048u)) mbar_wait(full0 + 8 * s, (kstep / K::ST) & 1);
        if (i == p1) mbar_wait(augf, it & 1);   // this unit's -L2/s is in B_aug
        if (mrec) mdbg[16384 + astep * 4 + 2] = gtimer();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async data -> tensor core
        tc_fence_after();
        const uint64_t kd0 = sw128_desc(smem_u32(Ks + s * K::STAGE_BYTES));
        const uint32_t dacc = tmem + a * 256;
        // descriptor start addresses are in 16-B units: a byte offset o adds o >> 4
        if (c.debug & 4u) {
          // debug: no MMA
        } else if (i < p1) {
#pragma unroll
          for (int half = 0; half < K::M1H; ++half)
#pragma unroll
            for (int k = 0; k < K::KSTEPS; ++k)
              umma_elect(dacc + half * 128, qd0 + (((k >> 2) * K::SLAB_Q + half * 128 * 128 + (k & 3) * 32) >> 4),
                         kd0 + (((k >> 2) * K::SLAB_K + (k & 3) * 32) >> 4), idesc_bf16(128, kTile), k > 0);
        } else {
#pragma unroll
          for (int k = 0; k < K::KSTEPS; ++k)
            umma_elect(dacc, kd0 + (((k >> 2) * K::SLAB_K + (k & 3) * 32) >> 4),
                       qd0 + (((k >> 2) * K::SLAB_Q + (k & 3) * 32) >> 4), idesc_bf16(kTile, K::GW), k > 0);
          umma_elect(dacc, aug_a, aug_b, idesc_bf16(kTile, K::GW), 1);
        }
        if (mrec) mdbg[16384 + astep * 4 + 3] = gtimer();
        umma_commit_elect(empty0 + 8 * s);   // K stage s free once these MMAs complete
        umma_commit_elect(accf0 + 8 * a);
      }
      umma_commit_elect(qempty0);            // Q buffer free once this unit's MMAs complete
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
    // ================= epilogue warps (8): two per TMEM lane quarter
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3;
    const int half = ew >> 2;
    const int col = half * 128 + q * 32 + lane;
    const bool warp_cols = (half * 128 + q * 32) < K::GW;
    const bool col_ok = col < K::GW;
    const int u1 = col_ok ? col / G : 0;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);

    // B_aug row of column c: (hi, mid, lo) bf16 with hi + mid + lo = -L2/s to ~2^-24 relative
    auto write_aug = [&](int cc, float L2) {
      const float nv = -L2 / scale;
      const __nv_bfloat16 hi = __float2bfloat16_rn(nv);
      const float r1 = nv - __bfloat162float(hi);
      const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
      const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
      const uint32_t w0 = (uint32_t)__bfloat16_as_ushort(hi) | ((uint32_t)__bfloat16_as_ushort(mid) << 16);
      const uint32_t w1 = (uint32_t)__bfloat16_as_ushort(lo);
      *reinterpret_cast<uint2*>(smem + K::OFF_AUG_B + (cc >> 3) * 256 + (cc & 7) * 16) = make_uint2(w0, w1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // visible to the tensor core
    };
    int astep = 0;
    // NEXT-4: caller's natural-log normaliser of this thread's column (u1, g) for a unit
    auto lse_input = [&](int un) {
      const int h = un % c.h_kv, l = (un / c.h_kv) % c.L, r = un / (c.h_kv * c.L);
      return __ldg(c.lse_in + (((size_t)l * c.M + c.q_slots[r]) * W + u1) * c.h_q + (size_t)h * G + (col - u1 * G));
    };
    float lse_next = 0.f;
    // debug timing (bit 1): [0] P1 step work, [2] P1 gap before step, [3] P2 ld, [4] P2 math, [5] P2 gap,
    // [1] P1 steps, [6] P2 work (start..end), [7] P2 steps
    uint32_t tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tlast = (uint32_t)gtimer();
    for (int it = 0, unit = cluster_id; unit < units; ++it, unit += nclusters) {
      const UnitInfo u = unit_info(unit);
      const int limit1 = u.T - W + u1;   // pass-1 causal limit of this column (R1, R2)
      float m = -INFINITY, ssum = 0.f, m1 = -INFINITY, s1 = 0.f;   // two pass-1 streams (see pair())
      for (int i = 0; i <= u.p1 + u.nt; ++i) {
        if (i == u.p1) {
          // ---- end of pass 1: LSE per column, combined across the cluster through DSMEM
          {   // merge the two streams into (m, ssum)
            const float mm = fmaxf(m, m1);
            const float mr = mm > -INFINITY ? mm : 0.f;
            ssum = ssum * ex2f(m - mr) + s1 * ex2f(m1 - mr);
            m = mm;
          }
          const int pb = it & 1;
          if (one_pass) {
            // NEXT-4: the normaliser of column (u, g) is the caller's natural-log LSE of query head
            // h*G + g at window row u; log2 domain like pass 1's
            // (the next unit's value is loaded here too, so its latency is off the next boundary)
            if (col_ok) {
              const float L2 = (it == 0 ? lse_input(u.id) : lse_next) * kLog2e;
              if (unit + nclusters < units) lse_next = lse_input(unit_info(unit + nclusters).id);
              write_aug(col, L2);
              if (rank == 0) c.ws.lse[(size_t)u.id * K::GW + col] = L2;
            }
          } else if (C == 1) {
            if (col_ok) {
              const float L2 = m + lg2f(ssum);
              write_aug(col, L2);
              c.ws.lse[(size_t)u.id * K::GW + col] = L2;
            }
          } else {
            if (col_ok) { pmv[pb * 256 + col] = m; psv[pb * 256 + col] = ssum; }
            named_bar(1, kEpiWarps * 32);
            if (ew == 0 && lane == 0) {
              asm volatile("fence.acq_rel.cluster;" ::: "memory");
#pragma unroll
              for (int rr = 0; rr < C; ++rr) mbar_remote_arrive(xchg0 + 8 * pb, rr);
            }
            mbar_wait_cluster(xchg0 + 8 * pb, (it >> 1) & 1);
            if (col_ok) {
              float M = -INFINITY, mr[C], sr[C];
#pragma unroll
              for (int rr = 0; rr < C; ++rr) {
                mr[rr] = ld_dsmem_f32(pmv + pb * 256 + col, rr);
                sr[rr] = ld_dsmem_f32(psv + pb * 256 + col, rr);
                M = fmaxf(M, mr[rr]);
              }
              float S = 0.f;
#pragma unroll
              for (int rr = 0; rr < C; ++rr)
                if (mr[rr] > -INFINITY) S += sr[rr] * ex2f(mr[rr] - M);
              const float L2 = M + lg2f(S);
              write_aug(col, L2);
              if (rank == 0) c.ws.lse[(size_t)u.id * K::GW + col] = L2;
            }
          }
          named_bar(1, kEpiWarps * 32);
          if (ew == 0 && lane == 0) mbar_arrive(augf);   // pass-2 MMAs of this unit may start
          if (i == u.p1 + u.nt) break;
          continue;
        }
        const int a = astep & 1;
        const bool rec = (c.debug & 1u) && blockIdx.x == 0 && ew == 0 && lane == 0 && astep < 1024;
        unsigned long long* dbg = reinterpret_cast<unsigned long long*>(c.ws.kept);
        if (rec) dbg[8192 + astep * 4 + 0] = gtimer();
        // MMA(astep) complete: each warp waits the commit mbarrier itself (try_wait parks the warp;
        // no cross-warp barrier, so warps are not held to the slowest one every step). No phase
        // aliasing: MMA(astep + 2) needs every epilogue warp's acc_empty arrival for astep.
        mbar_wait_lean(accf0 + 8 * a, (astep >> 1) & 1);
        if (rec) dbg[8192 + astep * 4 + 1] = gtimer();
        const uint32_t ts0 = (c.debug & 1u) ? (uint32_t)gtimer() : 0u;   // per-warp register timing (mod 2^32)
        if (c.debug & 1u) { tacc[(i < u.p1 ? 0 : 3) + 2] += ts0 - tlast; }
        tc_fence_after();
        if ((c.debug & 1u) && blockIdx.x == 0 && ew == 0 && lane == 0 && astep < 512)
          reinterpret_cast<unsigned long long*>(c.ws.kept)[astep * 4 + 2] = gtimer();
        const int t0 = tile_of(u, i < u.p1 ? i : i - 1) * kTile;
        if (c.debug & 2u) {
          // debug: no epilogue math
          __syncwarp();
          if (lane == 0) mbar_arrive(acce0 + 8 * a);
        } else if (i < u.p1) {
          // ---- pass 1: this thread owns window column `col`; 128 token logits in TMEM, consumed
          //      as 4 batches of 32 with the next batch's TMEM load in flight during the math. The
          //      batch loop stays rolled (ping-pong pairs) so its body fits the L0 instruction cache.
          // Two independent online (max, sum) streams per column -- even 32-token batches into
          // (m0, s0), odd ones into (m1, s1), merged at the end of pass 1 -- so each 64-token pair
          // carries two exp2 chains with no dependence between them (the MUFU pipe is fed from
          // both); the next pair's TMEM load is in flight during the math.
          constexpr int NB = 32;
          float vp[2 * NB];
          const uint32_t tbase_addr = lane_base + a * 256 + half * 128;
          // the causal limit only bites in the last tile(s) of a unit: a warp-uniform test per step
          // selects the masking variant, so the hot variant has no per-element compare or branch
          const bool need_mask = t0 + kTile - 1 > u.T - W;
          auto online = [&](const float* v, float& mm, float& ss) {
            // batch max as a depth-4 tree of 3-input FMNMX (a linear chain is 16 deep)
            float t3[11];
#pragma unroll
            for (int j = 0; j < 10; ++j) t3[j] = max3f(v[3 * j], v[3 * j + 1], v[3 * j + 2]);
            t3[10] = fmaxf(v[30], v[31]);
            const float mx = fmaxf(max3f(max3f(t3[0], t3[1], t3[2]), max3f(t3[3], t3[4], t3[5]),
                                         max3f(t3[6], t3[7], t3[8])),
                                   fmaxf(t3[9], t3[10]));
            const float mn = fmaxf(mm, mx * scale);             // -inf only if nothing valid yet
            const float mref = mn > -INFINITY ? mn : 0.f;
            const float rescale = ex2f(mm - mref);              // mm = -inf -> 0 (ss is 0 anyway)
            const float bsum = sum_exp_n<NB, ZPC_POLY_TC>(v, scale, mref);
            ss = ss * rescale + bsum;
            mm = mn;
          };
          // one 64-token pair: load, wait, two independent exp2 chains (the second warp of the SMSP
          // covers the load latency)
          auto pair = [&](int bp, auto mask_tag) {
            constexpr bool kMask = decltype(mask_tag)::value;
#pragma unroll
            for (int k = 0; k < 4; ++k) TMEM_LD16(tbase_addr + bp * 2 * NB + k * 16, vp, k * 16);
            tmem_wait_ld();
            if (bp + 1 == kTile / (2 * NB)) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(acce0 + 8 * a);
            }
            if constexpr (kMask) {
              const int tbase = t0 + bp * 2 * NB;
#pragma unroll
              for (int j = 0; j < 2 * NB; ++j) vp[j] = (tbase + j > limit1) ? -INFINITY : vp[j];
            }
            online(vp, m, ssum);
            online(vp + NB, m1, s1);
          };
          // warp-uniform: G*w = 32*G, so a warp's 32 columns are all valid or all padding
          if (!warp_cols) {
            // padding warp (columns >= G*w): only the accumulator release
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acce0 + 8 * a);
          } else if (!need_mask) {
#pragma unroll 1
            for (int bp = 0; bp < kTile / (2 * NB); ++bp) pair(bp, std::false_type{});
          } else {
#pragma unroll 1
            for (int bp = 0; bp < kTile / (2 * NB); ++bp) pair(bp, std::true_type{});
          }
        } else {
          // ---- pass 2: this thread owns token t and the W/2 window rows of its half. The MMA
          //      already subtracted L2/s (B_aug), so each row is max over its G heads, one FMUL,
          //      one exp2: S[t] = (1/w) sum_u 2^(s * max_g (q_ug.k_t - L2_ug/s))  (Alg. 2 / Eq. 3)
          const int t = t0 + q * 32 + lane;
          const int du = t - (u.T - W) - half * (W / 2);   // row uu of this half is causal iff uu >= du
          float v[K::HC];
#pragma unroll
          for (int k = 0; k < K::HC / 16; ++k) TMEM_LD16(lane_base + a * 256 + half * K::HC + k * 16, v, k * 16);
          tmem_wait_ld();
          const uint32_t ts1 = (c.debug & 1u) ? (uint32_t)gtimer() : 0u;
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acce0 + 8 * a);       // accumulator free for MMA(astep + 2)
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int uu = 0; uu < W / 2; ++uu) {
            const float* y = v + uu * G;
            float mx;
            if constexpr (G == 4) mx = fmaxf(max3f(y[0], y[1], y[2]), y[3]);
            else if constexpr (G == 5) mx = max3f(max3f(y[0], y[1], y[2]), y[3], y[4]);
            else if constexpr (G == 7) mx = max3f(max3f(y[0], y[1], y[2]), max3f(y[3], y[4], y[5]), y[6]);
            else if constexpr (G == 8) mx = max3f(max3f(y[0], y[1], y[2]), max3f(y[3], y[4], y[5]), fmaxf(y[6], y[7]));
            else {
              mx = y[0];
#pragma unroll
              for (int g = 1; g < G; ++g) mx = fmaxf(mx, y[g]);
            }
            const float pterm = ex2f(mx * scale);
            acc[uu & 3] += (uu >= du) ? pterm : 0.f;
          }
          const float accs = (acc[0] + acc[1]) + (acc[2] + acc[3]);
          float* cb = comb + (astep & 1) * kTile;
          if (half == 1) cb[q * 32 + lane] = accs;
          if (c.debug & 1u) { const uint32_t ts2 = (uint32_t)gtimer(); tacc[3] += ts1 - ts0; tacc[4] += ts2 - ts1; }
          named_bar(1, kEpiWarps * 32);
          if (half == 0 && t < u.T && !(c.debug & 16384u))
            c.ws.scores[(size_t)u.id * c.max_seq_len + t] = (accs + cb[q * 32 + lane]) * (1.0f / W);
        }
        if (rec) dbg[8192 + astep * 4 + 2] = gtimer();
        if (c.debug & 1u) {
          const uint32_t te = (uint32_t)gtimer();
          if (i < u.p1) { tacc[0] += te - ts0; tacc[1] += 1; } else { tacc[6] += te - ts0; tacc[7] += 1; }
          tlast = te;
        }
        ++astep;
      }
    }
    if ((c.debug & 1u) && lane == 0) {   // per-warp, per-CTA totals (cycles) -> kept[65536 + (cta*8 + ew)*8 + k]
      unsigned long long* out = reinterpret_cast<unsigned long long*>(c.ws.kept) + 65536 + ((size_t)blockIdx.x * 8 + ew) * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k) out[k] = tacc[k];
    }
  }
  // ---- teardown
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  if (C > 1) cluster_sync_all();   // no CTA leaves while a peer may still read its partials
}

// ------------------------------------------------------------------ overlapped two-pass kernel
// Same arithmetic as k_score_tc (pass 1: per-column online (max, sum); pass 2: max over the GQA
// group of the normalised logits, exp2, mean over the window), but the two passes of DIFFERENT units
// run interleaved on each SM: "super-unit" j issues pass 1 of unit j and pass 2 of unit j-1
// alternately, tile by tile, so the MUFU-bound pass-1 epilogue of one unit overlaps the tensor-core
// and K-gather work of the other's pass 2 (in k_score_tc they alternate per unit, leaving the tensor
// pipe idle during pass 1 and the MUFU idle during pass 2). Costs: two Q buffers (unit j's as the
// pass-1 A operand, unit j-1's as the pass-2 B operand), so the K ring has fewer stages.
// Handshakes (all ping-pong, so no mbarrier phase can alias):
//   qfull[b]/qempty[b]  Q producer <-> MMA   (buffer b = unit & 1; released after the unit's pass 2)
//   augf / auge         epilogue  <-> MMA   (B_aug holds one unit's -L2/s; written at the end of the
//                                            unit's pass 1, released by the commit after its pass 2)
//   accf[a]/acce[a], full[s]/empty[s]       as in k_score_tc
// 24 warps: producers as k_score_tc (0-7), pass-1 epilogue (8-15), pass-2 epilogue (16-23);
// registers: launch 80/thread (65536 / 768), producers -> 56, pass-1 warps -> 104, pass-2 warps keep 80
constexpr int kThreadsO = 768;
constexpr int kProdRegsO = 56;
constexpr int kP1RegsO = 104;
static_assert(8 * kProdRegsO + 8 * kP1RegsO + 8 * 80 <= 2048, "register file: 65536 = 32 lanes x 2048");

template <int G, int W, int D, int C>
struct CfgO {
  static constexpr int GW = G * W;
  static constexpr int M1H = (GW + 127) / 128;
  static constexpr int SLABS = D / 64;
  static constexpr int KSTEPS = D / 16;
  static constexpr int HC = (W / 2) * G;
  static constexpr uint32_t SLAB_Q = GW * 128;
  static constexpr uint32_t Q_BYTES = SLAB_Q * SLABS;
  static constexpr uint32_t SLAB_K = kTile * 128;
  static constexpr uint32_t STAGE_BYTES = kTile * D * 2;
  static constexpr uint32_t AUG_A_BYTES = kTile * 32;
  static constexpr uint32_t AUG_B_BYTES = GW * 32;
  static constexpr uint32_t OFF_Q0 = 0;
  static constexpr uint32_t OFF_Q1 = Q_BYTES;
  static constexpr uint32_t OFF_AUG_A = 2 * Q_BYTES;
  static constexpr uint32_t OFF_AUG_B = OFF_AUG_A + AUG_A_BYTES;
  static constexpr uint32_t AUG_END = (OFF_AUG_B + AUG_B_BYTES + 1023) / 1024 * 1024;
  static constexpr uint32_t F_BYTES = (4 * GW + 2 * kTile + 2 * 128) * 4;   // pmv[2][GW], psv[2][GW], comb[2][kTile], pmh[2][128]
  static constexpr uint32_t IDS_BYTES = kIdSlots * kMaxIds * 4;
  static constexpr uint32_t BAR_BYTES = 40 * 8 + 16;
  static constexpr uint32_t MISC = F_BYTES + IDS_BYTES + BAR_BYTES;
  static constexpr int STAGES_FIT = (int)((227 * 1024 - 1024 - MISC - AUG_END) / STAGE_BYTES);
  static constexpr int ST = STAGES_FIT > 6 ? 6 : STAGES_FIT;
  static constexpr uint32_t OFF_K = AUG_END;
  static constexpr uint32_t OFF_F = OFF_K + ST * STAGE_BYTES;
  static constexpr uint32_t OFF_IDS = OFF_F + F_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_IDS + IDS_BYTES;
  static constexpr uint32_t SMEM = OFF_BAR + BAR_BYTES + 1024;   // + alignment slack
  static_assert(GW % 32 == 0 && GW <= 256, "pass-2 UMMA N = G*w must be a multiple of 32, <= 256");
  static_assert(W == 32 || W == 16, "epilogue batching assumes w = 32 or 16");
  static_assert(ST >= 2, "K ring needs >= 2 stages");
  static_assert(Q_BYTES % 1024 == 0, "Q slabs must stay 1024-B aligned for SW128");
};

template <int G, int W, int D, int C>
__global__ void __launch_bounds__(kThreadsO, 1) k_score_ovl(Call c, const __grid_constant__ CUtensorMap tmap_q) {
  using K = CfgO<G, W, D, C>;
  if (*c.status != ZPC_OK) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Ks = smem + K::OFF_K;
  float* pmv = reinterpret_cast<float*>(smem + K::OFF_F);   // [2][GW] partial max (by unit parity)
  float* psv = pmv + 2 * K::GW;                               // [2][GW] partial sums
  float* comb = psv + 2 * K::GW;                              // [2][kTile] pass-2 half sums
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + K::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 40);
  int* ids = reinterpret_cast<int*>(smem + K::OFF_IDS);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + 8);
  // accumulators: 0, 1 = pass-1 sub-step buffers (64 tokens x 2 M-halves = 128 TMEM columns each),
  // 2 = pass 2 (G*w columns at 256)
  const uint32_t accf0 = smem_u32(bars + 16), acce0 = smem_u32(bars + 19);
  const uint32_t qfull0 = smem_u32(bars + 22), qempty0 = smem_u32(bars + 24);
  const uint32_t xchg0 = smem_u32(bars + 26);
  const uint32_t augf = smem_u32(bars + 28), auge = smem_u32(bars + 29);
  static_assert(K::ST <= 8, "barrier block holds 8 stages");

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int rank = C > 1 ? (int)(blockIdx.x % C) : 0;
  const int cluster_id = blockIdx.x / C;
  const int nclusters = gridDim.x / C;
  const int units = c.R * c.L * c.h_kv;
  const int nu = units > cluster_id ? (units - cluster_id + nclusters - 1) / nclusters : 0;   // units of this cluster

  if (threadIdx.x == 0) {
    for (int s = 0; s < K::ST; ++s) { mbar_init(full0 + 8 * s, kLoadWarps * 32); mbar_init(empty0 + 8 * s, 1); }
    for (int a = 0; a < 3; ++a) {
      mbar_init(accf0 + 8 * a, 1);
      mbar_init(acce0 + 8 * a, kEpiWarps);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(qfull0 + 8 * a, 1);
      mbar_init(qempty0 + 8 * a, 1);
      mbar_init(xchg0 + 8 * a, C);
    }
    mbar_init(augf, 1);
    mbar_init(auge, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_q)));
  {
    uint4* aug = reinterpret_cast<uint4*>(smem + K::OFF_AUG_A);
    for (int i = threadIdx.x; i < (int)((K::AUG_A_BYTES + K::AUG_B_BYTES) / 16); i += kThreadsO) {
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (i < (int)(K::AUG_A_BYTES / 16) && ((i >> 3) & 1) == 0) v = make_uint4(0x3F803F80u, 0x00003F80u, 0u, 0u);
      aug[i] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (C > 1) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const float scale = kLog2e * rsqrtf((float)D);

  struct UnitInfo { int r, l, h, T, slot, tb, nt; };
  auto unit_info = [&](int j) {   // j-th unit of this cluster
    const int unit = cluster_id + j * nclusters;
    UnitInfo u;
    u.h = unit % c.h_kv;
    u.l = (unit / c.h_kv) % c.L;
    u.r = unit / (c.h_kv * c.L);
    u.T = c.seq_lens[u.r];
    u.slot = c.q_slots[u.r];
    const int ntot = (u.T + kTile - 1) / kTile;
    u.tb = (int)((long long)ntot * rank / C);
    u.nt = (int)((long long)ntot * (rank + 1) / C) - u.tb;
    return u;
  };
  // step cursor over the interleaved schedule: super-unit j = pass 1 of unit j (slot 0) and pass 2
  // of unit j-1 (slot 1), alternating per pair index k; pass 1 ascending, pass 2 descending tiles
  struct Cur { int j, k, sub, nA, nB; UnitInfo A, B; };
  auto cur_init = [&](Cur& s) {
    s.j = 0; s.k = 0; s.sub = 0; s.nB = 0; s.nA = 0;
    if (nu > 0) { s.A = unit_info(0); s.nA = s.A.nt; }
  };
  auto cur_settle = [&](Cur& s) -> bool {   // move to the first valid step at or after (j, k, sub)
    while (true) {
      if (s.j > nu) return false;
      if (s.k >= max(s.nA, s.nB)) {
        if (++s.j > nu) return false;
        s.B = s.A; s.nB = s.nA; s.nA = 0;
        if (s.j < nu) { s.A = unit_info(s.j); s.nA = s.A.nt; }
        s.k = 0; s.sub = 0;
        continue;
      }
      if (s.sub == 0) { if (s.k < s.nA) return true; s.sub = 1; }
      if (s.k < s.nB) return true;
      s.sub = 0; ++s.k;
    }
  };
  auto cur_advance = [](Cur& s) { if (s.sub == 0) s.sub = 1; else { s.sub = 0; ++s.k; } };
  auto cur_tile = [](const Cur& s) { return s.sub == 0 ? s.A.tb + s.k : s.B.tb + s.B.nt - 1 - s.k; };

  if (warp < kEpiWarp0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegsO));
    if (warp == 0) {
      // ================= Q producer: unit j -> buffer j & 1, reloaded once unit j-2's pass 2 is done
      if (lane == 0) {
        const uint64_t drop = policy_evict_first();
        for (int j = 0; j < nu; ++j) {
          const UnitInfo u = unit_info(j);
          const int qb = j & 1;
          mbar_wait_backoff(qempty0 + 8 * qb, ((j >> 1) & 1) ^ 1, 2000);
          mbar_expect_tx(qfull0 + 8 * qb, K::Q_BYTES);
          const uint32_t qdst = smem_u32(smem + (qb ? K::OFF_Q1 : K::OFF_Q0));
          const int qrow = (u.l * c.M + u.slot) * W;
          for (int sl = 0; sl < K::SLABS; ++sl)
            tma_load_3d(qdst + sl * K::SLAB_Q, &tmap_q, sl * 64, u.h * G, qrow, qfull0 + 8 * qb, drop);
        }
      }
      __syncwarp();
    } else if (warp >= 3 && warp < 4 + kLoadWarps && (c.debug & 2048u)) {
      // bisection (ZPC_SCORE_DEBUG): no K gather, no feeder
    } else if (warp >= 4 && warp < 4 + kLoadWarps) {
      // ---- K gather (as k_score_tc): 16-B cp.async per thread into the SW128 K-major stage
      constexpr int CPR = D / 8;
      constexpr int RPP = kLoadWarps * 32 / CPR;
      static_assert(RPP % 8 == 0, "the per-thread SW128 swizzle term needs rows-per-pass % 8 == 0");
      const int et = threadIdx.x - 4 * 32;
      const int cr = et % CPR, rsub = et / CPR;
      const uint32_t chunk_off = (uint32_t)(cr >> 3) * K::SLAB_K;
      const uint16_t* Kg = reinterpret_cast<const uint16_t*>(c.k_cache);
      const uint32_t ids_base = smem_u32(ids);
      const bool b_pow2 = (c.b & (c.b - 1)) == 0;
      const int b_log2 = 31 - __clz(c.b);
      const uint32_t dst_thr = (uint32_t)rsub * 128u + (uint32_t)(((cr & 7) ^ (rsub & 7)) << 4) + chunk_off;
      const uint32_t hD = (uint32_t)c.h_kv * D;
      Cur s;
      cur_init(s);
      for (int ld_step = 0; cur_settle(s); ++ld_step, cur_advance(s)) {
        const UnitInfo& u = s.sub ? s.B : s.A;
        const int st = ld_step % K::ST;
        const int t0 = cur_tile(s) * kTile;
        const int j0 = b_pow2 ? (t0 >> b_log2) : t0 / c.b;
        const int T = u.T;
        const uint16_t* lbase = Kg + (size_t)u.l * c.N_total * c.b * hD + (size_t)u.h * D + cr * 8;
        const uint32_t dst0 = smem_u32(Ks + st * K::STAGE_BYTES) + dst_thr;
        named_bar(4, kLoadWarps * 32 + 32);                     // feeder: ids of this tile, stage free
        const uint32_t sid = ids_base + (uint32_t)(ld_step % kIdSlots) * kMaxIds * 4;
        if (c.b == 16) {
          constexpr int RB = 16 / RPP;
          constexpr int NBLK = kTile / 16;
          const uint32_t qstride = (uint32_t)RPP * hD;
          const uint32_t rbase = (uint32_t)rsub * hD;
          int blk[NBLK];
#pragma unroll
          for (int jb = 0; jb < NBLK; ++jb) {
            blk[jb] = lds_s32(sid + 4u * (uint32_t)jb);
            ZPC_CHECK(t0 + jb * 16 >= T || (blk[jb] >= 0 && blk[jb] < c.N_total));
          }
          if (t0 + kTile <= T) {
#pragma unroll
            for (int jb = 0; jb < NBLK; ++jb) {
              uint32_t off = (uint32_t)blk[jb] * 16u * hD + rbase;
#pragma unroll
              for (int q = 0; q < RB; ++q, off += qstride)
                cp_async16(dst0 + (uint32_t)((jb * 16 + q * RPP) * 128), lbase + off);
            }
          } else {
#pragma unroll
            for (int jb = 0; jb < NBLK; ++jb) {
              uint32_t off = (uint32_t)blk[jb] * 16u * hD + rbase;
#pragma unroll
              for (int q = 0; q < RB; ++q, off += qstride)
                if (t0 + jb * 16 + q * RPP + rsub < T)
                  cp_async16(dst0 + (uint32_t)((jb * 16 + q * RPP) * 128), lbase + off);
            }
          }
        } else {
          uint32_t off[kTile / RPP];
#pragma unroll
          for (int k = 0; k < kTile / RPP; ++k) {
            const int t = t0 + RPP * k + rsub;
            const int jr = b_pow2 ? (t >> b_log2) : t / c.b;
            const int blk = lds_s32(sid + 4u * (uint32_t)min(max(jr - j0, 0), kMaxIds - 1));
            ZPC_CHECK(t >= T || (blk >= 0 && blk < c.N_total && t - jr * c.b < c.b));
          off[k] = ((uint32_t)blk * (uint32_t)c.b + (uint32_t)(t - jr * c.b)) * hD;
          }
#pragma unroll
          for (int k = 0; k < kTile / RPP; ++k)
            if (t0 + RPP * k + rsub < T) cp_async16(dst0 + (uint32_t)(RPP * k * 128), lbase + off[k]);
        }
        cp_async_arrive_noinc(full0 + 8 * st);
      }
    } else if (warp == 3) {
      // ================= feeder (as k_score_tc): block ids kIdAhead tiles ahead + stage release
      static_assert(kIdSlots >= kIdAhead + 2, "id ring too small for the lookahead");
      Cur ls, ps;
      cur_init(ls);
      cur_init(ps);
      const uint32_t ids_base = smem_u32(ids);
      auto issue_ids = [&](int slot) {
        if (cur_settle(ls)) {
          const UnitInfo& u = ls.sub ? ls.B : ls.A;
          const int t0 = cur_tile(ls) * kTile;
          const int j0 = t0 / c.b;
          const int nb = (min(t0 + kTile, u.T) - 1) / c.b - j0 + 1;
          if (lane < nb)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ids_base + (uint32_t)(slot * kMaxIds + lane) * 4u),
                         "l"(c.tables + (size_t)u.r * c.table_stride + j0 + lane) : "memory");
          cur_advance(ls);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
#pragma unroll 1
      for (int k = 0; k < kIdAhead; ++k) issue_ids(k);
      for (int g = 0; cur_settle(ps); ++g, cur_advance(ps)) {
        issue_ids((g + kIdAhead) % kIdSlots);
        if (g >= K::ST) {
          if (lane == 0) mbar_wait(empty0 + 8 * (g % K::ST), ((g / K::ST) & 1) ^ 1);
          __syncwarp();
        }
        asm volatile("cp.async.wait_group %0;" ::"n"(kIdAhead) : "memory");
        named_bar(4, kLoadWarps * 32 + 32);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp == 1) {
      // ================= MMA issuer (converged warp, elected lane issues)
      int kstep = 0, n1 = 0, n2 = 0;   // K stages issued; pass-1 / pass-2 steps issued
      const uint64_t aug_a = none_desc(smem_u32(smem + K::OFF_AUG_A), 128, 256);
      const uint64_t aug_b = none_desc(smem_u32(smem + K::OFF_AUG_B), 128, 256);
      const uint64_t qd0 = sw128_desc(smem_u32(smem + K::OFF_Q0));
      const uint64_t qd1 = sw128_desc(smem_u32(smem + K::OFF_Q1));
      int nA = 0, nB = 0;
      for (int j = 0; j <= nu; ++j) {
        nB = nA;
        nA = 0;
        if (j < nu) nA = __shfl_sync(0xffffffffu, unit_info(j).nt, 0);
        const uint64_t qdA = (j & 1) ? qd1 : qd0, qdB = (j & 1) ? qd0 : qd1;
        bool q_ok = j >= nu, aug_ok = j == 0;
        // a part with no steps waits its handshake up front (keeps the ping-pong strict)
        if (!q_ok && nA == 0) { mbar_wait(qfull0 + 8 * (j & 1), (j >> 1) & 1); q_ok = true; }
        if (!aug_ok && nB == 0) { mbar_wait(augf, (j - 1) & 1); aug_ok = true; }
        const int np = max(nA, nB);
        for (int k = 0; k < np; ++k) {
#pragma unroll 1
          for (int sub = 0; sub < 2; ++sub) {
            if (sub == 0 ? k >= nA : k >= nB) continue;
            const int s = kstep % K::ST;
            if (!(c.debug & 2048u)) mbar_wait(full0 + 8 * s, (kstep / K::ST) & 1);
            if (sub == 0 && !q_ok) { mbar_wait(qfull0 + 8 * (j & 1), (j >> 1) & 1); q_ok = true; }
            if (sub == 1 && !aug_ok) { mbar_wait(augf, (j - 1) & 1); aug_ok = true; }
            const uint64_t kd0 = sw128_desc(smem_u32(Ks + s * K::STAGE_BYTES));
            if (sub == 0) {
              // pass 1: two 64-token sub-steps, each into its own double-buffered accumulator, so the
              // epilogue frees a buffer right after loading it (N = 64; B = rows 64*hs.. of the stage)
#pragma unroll 1
              for (int hs = 0; hs < (K::M1H == 1 ? 1 : 2); ++hs, ++n1) {
                const int a = n1 & 1;
                mbar_wait(acce0 + 8 * a, ((n1 >> 1) & 1) ^ 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tc_fence_after();
                const uint32_t dacc = tmem + a * 128;
                if (K::M1H == 1) {
                  // one M-half: the whole 128-token tile in one sub-step (N = 128, 128 columns)
                  if (!(c.debug & 4u)) {
#pragma unroll
                    for (int kk = 0; kk < K::KSTEPS; ++kk)
                      umma_elect(dacc, qdA + (((kk >> 2) * K::SLAB_Q + (kk & 3) * 32) >> 4),
                                 kd0 + (((kk >> 2) * K::SLAB_K + (kk & 3) * 32) >> 4), idesc_bf16(128, kTile), kk > 0);
                  }
                } else if (!(c.debug & 4u)) {
#pragma unroll
                  for (int half = 0; half < K::M1H; ++half)
#pragma unroll
                    for (int kk = 0; kk < K::KSTEPS; ++kk)
                      umma_elect(dacc + half * 64,
                                 qdA + (((kk >> 2) * K::SLAB_Q + half * 128 * 128 + (kk & 3) * 32) >> 4),
                                 kd0 + (((kk >> 2) * K::SLAB_K + hs * 64 * 128 + (kk & 3) * 32) >> 4),
                                 idesc_bf16(128, 64), kk > 0);
                }
                umma_commit_elect(accf0 + 8 * a);
              }
            } else {
              mbar_wait(acce0 + 16, (n2 & 1) ^ 1);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              tc_fence_after();
              const uint32_t dacc = tmem + 256;
              if (!(c.debug & 4u)) {
#pragma unroll
                for (int kk = 0; kk < K::KSTEPS; ++kk)
                  umma_elect(dacc, kd0 + (((kk >> 2) * K::SLAB_K + (kk & 3) * 32) >> 4),
                             qdB + (((kk >> 2) * K::SLAB_Q + (kk & 3) * 32) >> 4), idesc_bf16(kTile, K::GW), kk > 0);
                umma_elect(dacc, aug_a, aug_b, idesc_bf16(kTile, K::GW), 1);
              }
              umma_commit_elect(accf0 + 16);
              ++n2;
            }
            umma_commit_elect(empty0 + 8 * s);
            ++kstep;
          }
        }
        if (j > 0) {
          umma_commit_elect(auge);                   // B_aug (unit j-1) free once its pass-2 MMAs complete
          umma_commit_elect(qempty0 + 8 * ((j - 1) & 1));   // and unit j-1's Q buffer
        }
      }
    }
  } else if (warp < kEpiWarp0 + 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kP1RegsO));
    // ================= pass-1 warps (8, two per TMEM lane quarter): column col = half*128 + q*32 + lane
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3;
    const int half = ew >> 2;
    const int col = half * 128 + q * 32 + lane;
    const bool col_ok = col < K::GW;
    // G*w <= 128 (one M-half): the two warps of a quarter share the columns and split each tile's
    // tokens (64 each, one N = 128 MMA per tile) instead of leaving the second warp idle
    constexpr bool kSplit = K::M1H == 1;
    constexpr int kSub = kSplit ? 1 : 2;           // pass-1 sub-steps (accumulator buffers) per tile
    const int pcol = kSplit ? q * 32 + lane : col;  // this thread's column in pass 1
    const bool warp_cols = (kSplit ? q * 32 : half * 128 + q * 32) < K::GW;
    const int u1 = pcol < K::GW ? pcol / G : 0;
    float* pmh = comb + 2 * kTile;                  // [2][128] split-half merge (m, s)
    const uint32_t tbase0 = tmem + ((uint32_t)(q * 32) << 16) + half * 64;   // + 128 * buffer
    auto write_aug = [&](int cc, float L2) {
      const float nv = -L2 / scale;
      const __nv_bfloat16 hi = __float2bfloat16_rn(nv);
      const float r1 = nv - __bfloat162float(hi);
      const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
      const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
      const uint32_t w0 = (uint32_t)__bfloat16_as_ushort(hi) | ((uint32_t)__bfloat16_as_ushort(mid) << 16);
      const uint32_t w1 = (uint32_t)__bfloat16_as_ushort(lo);
      *reinterpret_cast<uint2*>(smem + K::OFF_AUG_B + (cc >> 3) * 256 + (cc & 7) * 16) = make_uint2(w0, w1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    };
    int n1 = 0;
    for (int j = 0; j < nu; ++j) {
      const UnitInfo A = unit_info(j);
      const int unitA = cluster_id + j * nclusters;
      const int limit1 = A.T - W + u1;                // pass-1 causal limit of this column (R1, R2)
      float m = -INFINITY, ssum = 0.f, m1 = -INFINITY, s1 = 0.f;
      for (int k = 0; k < A.nt; ++k) {
        if (c.debug & 2u) {   // bisection: no epilogue math
          for (int hs = 0; hs < kSub; ++hs, ++n1) {
            mbar_wait(accf0 + 8 * (n1 & 1), (n1 >> 1) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(acce0 + 8 * (n1 & 1));
          }
          continue;
        }
        // two online (max, sum) streams per column (as k_score_tc)
        const int t0 = (A.tb + k) * kTile;
        constexpr int NB = 32;
        float vp[2 * NB];
        const bool need_mask = t0 + kTile - 1 > A.T - W;
        auto online = [&](const float* v, float& mm, float& ss) {
          float t3[11];
#pragma unroll
          for (int jj = 0; jj < 10; ++jj) t3[jj] = max3f(v[3 * jj], v[3 * jj + 1], v[3 * jj + 2]);
          t3[10] = fmaxf(v[30], v[31]);
          const float mx = fmaxf(max3f(max3f(t3[0], t3[1], t3[2]), max3f(t3[3], t3[4], t3[5]),
                                       max3f(t3[6], t3[7], t3[8])),
                                 fmaxf(t3[9], t3[10]));
          const float mn = fmaxf(mm, mx * scale);
          const float mref = mn > -INFINITY ? mn : 0.f;
          const float rescale = ex2f(mm - mref);
          const float bsum = sum_exp_n<NB, kSplit ? ZPC_POLY_SPLIT : kPolyEighths>(v, scale, mref);
          ss = ss * rescale + bsum;
          mm = mn;
        };
        // one 64-token sub-step: wait its MMA, load, free the buffer, then the math
        auto pair = [&](int bp, auto mask_tag) {
          constexpr bool kMask = decltype(mask_tag)::value;
          const int a = n1 & 1;
          mbar_wait_lean(accf0 + 8 * a, (n1 >> 1) & 1);
          tc_fence_after();
          ++n1;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) TMEM_LD16(tbase0 + a * 128 + kk * 16, vp, kk * 16);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acce0 + 8 * a);
          if constexpr (kMask) {
            const int tb = t0 + (kSplit ? half : bp) * 2 * NB;
#pragma unroll
            for (int jj = 0; jj < 2 * NB; ++jj) vp[jj] = (tb + jj > limit1) ? -INFINITY : vp[jj];
          }
          online(vp, m, ssum);
          online(vp + NB, m1, s1);
        };
        if (!warp_cols) {
          for (int hs = 0; hs < kSub; ++hs, ++n1) {
            mbar_wait_lean(accf0 + 8 * (n1 & 1), (n1 >> 1) & 1);
            tc_fence_after();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acce0 + 8 * (n1 & 1));
          }
        } else if (!need_mask) {
#pragma unroll 1
          for (int bp = 0; bp < kSub; ++bp) pair(bp, std::false_type{});
        } else {
#pragma unroll 1
          for (int bp = 0; bp < kSub; ++bp) pair(bp, std::true_type{});
        }
      }
      // ---- end of unit A's pass 1: LSE per column (cluster-combined), into B_aug once the previous
      //      unit's pass-2 MMAs released it
      {
        const float mm = fmaxf(m, m1);
        const float mr = mm > -INFINITY ? mm : 0.f;
        ssum = ssum * ex2f(m - mr) + s1 * ex2f(m1 - mr);
        m = mm;
      }
      if constexpr (kSplit) {   // fold the second token half into the first warp of the quarter
        if (half == 1) { pmh[q * 32 + lane] = m; pmh[128 + q * 32 + lane] = ssum; }
        named_bar(1, 8 * 32);
        if (half == 0) {
          const float mo = pmh[q * 32 + lane], so = pmh[128 + q * 32 + lane];
          const float mm = fmaxf(m, mo);
          const float mr = mm > -INFINITY ? mm : 0.f;
          ssum = ssum * ex2f(m - mr) + so * ex2f(mo - mr);
          m = mm;
        }
      }
      float L2 = 0.f;
      if (C == 1) {
        if (col_ok) L2 = m + lg2f(ssum);
      } else {
        const int pb = j & 1;
        if (col_ok) { pmv[pb * K::GW + col] = m; psv[pb * K::GW + col] = ssum; }
        named_bar(1, 8 * 32);
        if (ew == 0 && lane == 0) {
          asm volatile("fence.acq_rel.cluster;" ::: "memory");
#pragma unroll
          for (int rr = 0; rr < C; ++rr) mbar_remote_arrive(xchg0 + 8 * pb, rr);
        }
        mbar_wait_cluster(xchg0 + 8 * pb, (j >> 1) & 1);
        if (col_ok) {
          float M = -INFINITY, mr[C], sr[C];
#pragma unroll
          for (int rr = 0; rr < C; ++rr) {
            mr[rr] = ld_dsmem_f32(pmv + pb * K::GW + col, rr);
            sr[rr] = ld_dsmem_f32(psv + pb * K::GW + col, rr);
            M = fmaxf(M, mr[rr]);
          }
          float S = 0.f;
#pragma unroll
          for (int rr = 0; rr < C; ++rr)
            if (mr[rr] > -INFINITY) S += sr[rr] * ex2f(mr[rr] - M);
          L2 = M + lg2f(S);
        }
      }
      mbar_wait(auge, (j & 1) ^ 1);   // pass-2 MMAs of unit j-1 (the last readers of B_aug) done
      if (col_ok) {
        write_aug(col, L2);
        if (rank == 0) c.ws.lse[(size_t)unitA * K::GW + col] = L2;
      }
      named_bar(1, 8 * 32);
      if (ew == 0 && lane == 0) mbar_arrive(augf);
    }
  } else {
    // ================= pass-2 warps (8, two per lane quarter): token t = t0 + q*32 + lane, window
    // rows [half*W/2, half*W/2 + W/2), read from accumulator 1 in chunks of 8 rows (8G columns).
    // The MMA already subtracted L2/s (B_aug): S[t] = (1/w) sum_u 2^(s * max_g (q_ug.k_t - L2_ug/s))
    const int ew = warp - kEpiWarp0 - 8;
    const int q = warp & 3;
    const int half = ew >> 2;
    const uint32_t tbase1 = tmem + ((uint32_t)(q * 32) << 16) + 256 + half * K::HC;   // accumulator 2
    constexpr int RC = G >= 7 ? 4 : 8;    // window rows per chunk (RC*G values in 80 registers)
    constexpr int NCH = (W / 2) / RC;     // chunks per half
    int n2 = 0;
    for (int j = 0; j < nu; ++j) {
      const UnitInfo B = unit_info(j);
      const int unitB = cluster_id + j * nclusters;
      for (int k = 0; k < B.nt; ++k, ++n2) {
        mbar_wait_lean(accf0 + 16, n2 & 1);
        tc_fence_after();
        const int t0 = (B.tb + B.nt - 1 - k) * kTile;
        const int t = t0 + q * 32 + lane;
        const int du = t - (B.T - W) - half * (W / 2);   // row uu of this half is causal iff uu >= du
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        if (c.debug & 2u) {
          __syncwarp();
          if (lane == 0) mbar_arrive(acce0 + 16);
          continue;
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          float v[RC * G];
#pragma unroll
          for (int kk = 0; kk < RC * G / 4; ++kk) TMEM_LD4(tbase1 + ch * RC * G + kk * 4, v, kk * 4);
          tmem_wait_ld();
          if (ch + 1 == NCH) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acce0 + 16);   // accumulator 1 free for the next pass-2 MMA
          }
#pragma unroll
          for (int r = 0; r < RC; ++r) {
            const float* y = v + r * G;
            float mx;
            if constexpr (G == 4) mx = fmaxf(max3f(y[0], y[1], y[2]), y[3]);
            else if constexpr (G == 5) mx = max3f(max3f(y[0], y[1], y[2]), y[3], y[4]);
            else if constexpr (G == 7) mx = max3f(max3f(y[0], y[1], y[2]), max3f(y[3], y[4], y[5]), y[6]);
            else if constexpr (G == 8) mx = max3f(max3f(y[0], y[1], y[2]), max3f(y[3], y[4], y[5]), fmaxf(y[6], y[7]));
            else {
              mx = y[0];
#pragma unroll
              for (int g = 1; g < G; ++g) mx = fmaxf(mx, y[g]);
            }
            const float pterm = ex2f(mx * scale);
            acc[r & 3] += (ch * RC + r >= du) ? pterm : 0.f;
          }
        }
        const float accs = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        float* cb = comb + (n2 & 1) * kTile;   // alternate per pass-2 step
        if (half == 1) cb[q * 32 + lane] = accs;
        named_bar(2, 8 * 32);
        if (half == 0 && t < B.T)
          c.ws.scores[(size_t)unitB * c.max_seq_len + t] = (accs + cb[q * 32 + lane]) * (1.0f / W);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  if (C > 1) cluster_sync_all();
}


// ------------------------------------------------------------------ host side

template <int G, int W, int D, int C, bool OVL>
cudaError_t launch_tc(const Call& c, const CUtensorMap& tq, cudaStream_t s) {
  using K = std::conditional_t<OVL, CfgO<G, W, D, C>, Cfg<G, W, D, C>>;
  auto kern = OVL ? k_score_ovl<G, W, D, C> : k_score_tc<G, W, D, C>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
  if (e != cudaSuccess) return e;
  if (C > 1) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
  const int units = c.R * c.L * c.h_kv;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(OVL ? kThreadsO : kThreads);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent: as many clusters as can be co-resident (one CTA per SM), each looping over units
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int max_clusters = sms / C;
  cfg.gridDim = dim3(C);
  int q = 0;
  if (cudaOccupancyMaxActiveClusters(&q, kern, &cfg) == cudaSuccess && q > 0) max_clusters = q;
  cudaGetLastError();
  cfg.gridDim = dim3((unsigned)(std::min(units, max_clusters) * C));
  return cudaLaunchKernelEx(&cfg, kern, c, tq);
}

// Cluster size: CTAs per unit. Splitting a unit's tokens over C CTAs shrinks the K slice each
// CTA re-reads in pass 2 (in flight across the GPU: ~148/C slices), keeping it L2-resident
// (DESIGN.md §Score kernel, L2 reuse). Tuning builds (-DZPC_TUNING) read ZPC_SCORE_CLUSTER (1/2/4/8).
int cluster_size(const Call& c) {
#ifdef ZPC_TUNING
  if (const char* e = getenv("ZPC_SCORE_CLUSTER")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8) return v;
  }
#endif
  return c.max_seq_len < 2 * kTile ? 1 : 2;
}

// Two-pass calls use the overlapped kernel (pass 1 of unit j || pass 2 of unit j-1); single-pass
// calls (ZPC_F_LSE_INPUT) have no pass 1 to overlap and keep k_score_tc's deeper K ring.
// Tuning builds read ZPC_SCORE_OVL=0 to select k_score_tc for two-pass calls too (same-box A/B runs).
bool use_ovl(const Call& c) {
  // w = 16 (the paper's b = 256 operating point, ~16 units per cluster per call): measured faster
  // serial (0.34 vs 0.46 ms per 4-request call), the interleave's start/drain is not amortised
  if (c.lse_in != nullptr || c.w == 16 || (c.variant & ZPC_V_SCORE_SERIAL)) return false;
#ifdef ZPC_TUNING
  if (const char* e = getenv("ZPC_SCORE_OVL")) return atoi(e) != 0;
#endif
  return true;
}

template <int G, int W, int D, bool OVL>
cudaError_t launch_o(const Call& c, const CUtensorMap& tq, cudaStream_t s) {
#ifdef ZPC_SCORE_BIG_CLUSTERS   // tuning builds only: 4- and 8-CTA clusters measured slower
  switch (cluster_size(c)) {
    case 8: return launch_tc<G, W, D, 8, OVL>(c, tq, s);
    case 4: return launch_tc<G, W, D, 4, OVL>(c, tq, s);
    default: break;
  }
#endif
  return cluster_size(c) >= 2 ? launch_tc<G, W, D, 2, OVL>(c, tq, s) : launch_tc<G, W, D, 1, OVL>(c, tq, s);
}

// OVL_OK: the overlapped two-pass instance exists for this shape. Two-pass w = 32 calls with G = 5, 7, 8
// are taken by the cooperative kernel (score_coop.cu) before this dispatcher; they arrive here only as
// single-pass (ZPC_F_LSE_INPUT) calls.
template <int G, int W, int D, bool OVL_OK>
cudaError_t launch_c(const Call& c, const CUtensorMap& tq, cudaStream_t s) {
  if constexpr (OVL_OK)
    if (use_ovl(c)) return launch_o<G, W, D, true>(c, tq, s);
  return launch_o<G, W, D, false>(c, tq, s);
}

template <int D>
cudaError_t dispatch_g(const Call& c, const CUtensorMap& tq, cudaStream_t s, bool* used) {
  if (c.w == 16 && D == 128) {
    // the paper's own operating point (w = 16): Qwen3-8B / DS-Llama-8B (G = 4), 32B (G = 8)
    *used = true;
    switch (c.G) {
      case 4: return launch_c<4, 16, D, false>(c, tq, s);
      case 8: return launch_c<8, 16, D, false>(c, tq, s);
      default: *used = false; return cudaSuccess;
    }
  }
  if (c.w != 32) return cudaSuccess;
  *used = true;
  switch (c.G) {
    // MHA (G = 1) and the other GQA ratios up to 8 (MQA and GQA in general)
    case 1: return launch_c<1, 32, D, false>(c, tq, s);
    case 2: return launch_c<2, 32, D, false>(c, tq, s);
    case 3: return launch_c<3, 32, D, false>(c, tq, s);
    case 4: return launch_c<4, 32, D, true>(c, tq, s);
    case 5: return launch_c<5, 32, D, false>(c, tq, s);
    case 6: return launch_c<6, 32, D, false>(c, tq, s);
    case 7: return launch_c<7, 32, D, false>(c, tq, s);
    case 8: return launch_c<8, 32, D, false>(c, tq, s);
    default: *used = false; return cudaSuccess;
  }
}

}  // namespace

bool score_tc_applies(const Call& c) {
  if (c.dtype != ZPC_BF16 || (c.d != 64 && c.d != 128) || c.b < 5) return false;
  if (c.w == 16) return c.d == 128 && (c.G == 4 || c.G == 8);
  return c.w == 32 && c.G >= 1 && c.G <= 8;
}

cudaError_t launch_score_tc(const Call& c_in, cudaStream_t s, bool* used) {
  *used = false;
  Call c = c_in;
#ifdef ZPC_TUNING   // bisection switches; the production library reads no environment
  if (const char* e = getenv("ZPC_SCORE_DEBUG")) c.debug = (uint32_t)strtoul(e, nullptr, 10);
#endif
  if (c.dtype != ZPC_BF16) return cudaSuccess;
  if (c.d != 64 && c.d != 128) return cudaSuccess;
  if (c.b < 5) return cudaSuccess;   // a 128-token tile must span <= kMaxIds blocks
  if (c.R * c.L * c.h_kv == 0) { *used = true; return cudaSuccess; }
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaSuccess;
  const cuuint32_t estr[3] = {1, 1, 1};
  // Q cache viewed as [rows = L*M*w][h_q][d]; one box = the unit's G heads x w window rows
  CUtensorMap tq;
  const cuuint64_t qdim[3] = {(cuuint64_t)c.d, (cuuint64_t)c.h_q, (cuuint64_t)c.L * c.M * c.w};
  const cuuint64_t qstr[2] = {(cuuint64_t)c.d * 2, (cuuint64_t)c.h_q * c.d * 2};
  const cuuint32_t qbox[3] = {64, (cuuint32_t)c.G, (cuuint32_t)c.w};
  if (enc(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(c.q_cache), qdim, qstr, qbox, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaSuccess;   // not expressible as a tensor map: CUDA-core path
  return c.d == 64 ? dispatch_g<64>(c, tq, s, used) : dispatch_g<128>(c, tq, s, used);
}

}  // namespace zpc
