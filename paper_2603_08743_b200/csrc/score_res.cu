// a1 + a2 for short units (the paper's operating point, b = 256, w = 16, T ~ N_max*b = 2304): every logit
// computed ONCE and kept in TMEM.
//
// What it computes (Alg. 1 + §C.2), per unit (request r, layer l, KV head h):
//   x[c,t] = q_c . k_t / sqrt(d)   for the G*w window columns c = u*G + g and tokens t < T,
//   LSE[c] = log sum_{t <= T-w+u} exp x[c,t]
//   S[t]   = (1/w) sum_{u: t <= T-w+u} exp(max_g (x[(u,g),t] - LSE[(u,g)]))
//
// Why ("k_score_res"): the two-pass kernels recompute every logit in pass 2 (a second MMA over a
// second read of K) because a unit's logits do not fit on chip. At the paper's operating point they do: a unit
// is T / 128 tiles of 128 tokens x G*w = 64 fp32 columns, and a C-CTA cluster holds C x 512 / (G*w) tiles in
// TMEM (C = 4: 32 tiles = 4096 tokens). So each CTA of the cluster gathers its slice of the unit's keys once,
// issues ONE tcgen05.mma per tile (A = K tile, M = 128 tokens; B = Q, N = G*w) into its own TMEM slot, and the
// epilogue sweeps the resident logits three times: (A) per-column max, (B) per-column sum of
// 2^(x*s - max) -- both reduced over the CTA's tokens, then exchanged as (max, sum) pairs through DSMEM and
// merged into LSE -- and (C) the scores. K is read from HBM once and the tensor core does one pass (the
// two-pass kernels: two reads and two MMAs). Slots are a ring: the next unit's tiles are gathered and
// multiplied into the free slots while the epilogue sweeps the current one.
//
// Warp roles (512 threads): 0 Q producer (TMA, double buffer), 1 MMA issuer, 3 feeder (block ids, stage
// release), 4-11 epilogue (two groups of one warp per lane quarter q = warp & 3, i.e. 32 tokens of a tile),
// 12-15 K gather (16-B cp.async into the SW128 K-major stage; highest warp ids, which the issue arbiter favours).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "internal.h"
#include "tc_util.h"

namespace zpc {
namespace {

constexpr int kRThreads = 512;
constexpr int kRLoadWarps = 4;
constexpr int kREpi0 = 4;     // epilogue warps 4..11; K gather warps 12..15 (the warp arbiter favours
                              // high warp ids: the gather must not starve behind the epilogue's sweeps)
constexpr int kRLoad0 = 12;
constexpr int kREpiWarps = 8;
constexpr int kRProdRegs = 72;
constexpr int kREpiRegs = 184;
static_assert(8 * kRProdRegs + 8 * kREpiRegs <= 2048, "register file: 65536 = 32 lanes x 2048");

template <int G, int W, int D, int C>
struct CfgR {
  static constexpr int GW = G * W;
  static constexpr int NCW = GW / 2;                    // columns per epilogue warp (its half of the window rows)
  static constexpr int NS = 512 / GW;                   // TMEM slots (one tile's GW columns each)
  static constexpr int SLABS = D / 64;
  static constexpr int KSTEPS = D / 16;
  static constexpr uint32_t SLAB_Q = GW * 128;
  static constexpr uint32_t Q_BYTES = SLAB_Q * SLABS;
  static constexpr uint32_t SLAB_K = kTile * 128;
  static constexpr uint32_t STAGE_BYTES = kTile * D * 2;
  // floats: per epilogue group red[4][GW], mloc[GW], L2[GW]; xbuf[2 groups][2 parities][C ranks][GW] float2
  static constexpr uint32_t F_FLOATS = 12 * GW + 2 * 2 * C * GW * 2 + 8 * GW + 4;   // + wref[2][4][GW], oflag[2]
  static constexpr uint32_t MISC = F_FLOATS * 4 + kIdSlots * kMaxIds * 4 + 64 * 8;
  static constexpr int STAGES_FIT = (int)((227 * 1024 - 2 * Q_BYTES - MISC) / STAGE_BYTES);
  static constexpr int ST = STAGES_FIT > 6 ? 6 : STAGES_FIT;
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = 2 * Q_BYTES;
  static constexpr uint32_t OFF_F = OFF_K + ST * STAGE_BYTES;
  static constexpr uint32_t OFF_IDS = OFF_F + F_FLOATS * 4;
  static constexpr uint32_t OFF_BAR = OFF_IDS + kIdSlots * kMaxIds * 4;
  static constexpr uint32_t SMEM = OFF_BAR + 64 * 8;
  static_assert(GW % 32 == 0 && GW <= 64, "a warp holds a tile's G*w columns of its 32 tokens in registers");
  static_assert(W % 2 == 0, "window rows split in two halves");
  static_assert(NS >= 2 && NS <= 16, "TMEM slot ring");
  static_assert(ST >= 2, "K ring depth");
  static_assert(Q_BYTES % 1024 == 0, "Q slabs must stay 1024-B aligned for SW128");
  static_assert(SMEM <= 227 * 1024, "dynamic shared memory per CTA");
};

// remote shared-memory store of (a, b) to the same offset in cluster rank `rank`, completing 8 bytes of that
// rank's mbarrier (at the same offset as local_bar): DSMEM push with no release fence
__device__ __forceinline__ void st_async_v2(uint32_t local_addr, uint32_t local_bar, int rank, float a, float b) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(local_bar), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
               ::"r"(ra), "f"(a), "f"(b), "r"(rb) : "memory");
}

// max over the group of G heads of y[0..G)
template <int G>
__device__ __forceinline__ float gmax(const float* y) {
  if constexpr (G == 4) return fmaxf(max3f(y[0], y[1], y[2]), y[3]);
  else if constexpr (G == 8) return max3f(max3f(y[0], y[1], y[2]), max3f(y[3], y[4], y[5]), fmaxf(y[6], y[7]));
  else {
    float m = y[0];
#pragma unroll
    for (int g = 1; g < G; ++g) m = fmaxf(m, y[g]);
    return m;
  }
}

// lane j of the warp ends with OP over the warp's 32 lanes of column j + 32k of v[] (k < N/32): a
// transposing butterfly (at each level a lane keeps one half of its columns and folds in the partner's
// copy of that half), N - 1 shuffles for N columns
template <int N, bool MAX>
__device__ __forceinline__ void warp_col_reduce(float* v, int lane) {
#pragma unroll
  for (int w = N / 2, o = 16; w >= N / 32 && o >= 1; w >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < w; ++j) {
      // columns are kept in v[0..w): lanes with bit o set keep the upper half, the others the lower
      const float keep = up ? v[j + w] : v[j];
      const float send = up ? v[j] : v[j + w];
      const float recv = __shfl_xor_sync(0xffffffffu, send, o);
      v[j] = MAX ? fmaxf(keep, recv) : keep + recv;
    }
  }
}
// after warp_col_reduce<N>: the columns lane `lane` holds, in v[0..N/32)
template <int N>
__device__ __forceinline__ int reduced_col(int lane, int k) {
  // level with partner o kept the upper half iff lane & o: bits of the lane (MSB first) index the column
  int c = 0;
#pragma unroll
  for (int o = 16, w = N / 2; o >= 1 && w >= N / 32; o >>= 1, w >>= 1)
    if (lane & o) c += w;
  return c + k;
}

// tuning builds: timestamps of cluster 0 / rank 0 into the kept workspace region (a score-only call)
#ifdef ZPC_TUNING
#define RTRACE(i, v) do { if ((c.debug & 1u) && blockIdx.x < C && (i) < 8192) \
    reinterpret_cast<unsigned long long*>(c.ws.kept)[blockIdx.x * 8192 + (i)] = (v); } while (0)
#else
#define RTRACE(i, v) do { } while (0)
#endif

template <int G, int W, int D, int C>
__global__ void __launch_bounds__(kRThreads, 1) k_score_res(Call c, const __grid_constant__ CUtensorMap tmap_q,
                                                           const __grid_constant__ CUtensorMap tmap_k, int ktma) {
  using K = CfgR<G, W, D, C>;
  if (*c.status != ZPC_OK) return;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();   // SW128 operands need the 1024-B aligned base
  uint8_t* Ks = smem + K::OFF_K;
  int* ids = reinterpret_cast<int*>(smem + K::OFF_IDS);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + K::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 62);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + 8);             // [ST]
  const uint32_t sfull0 = smem_u32(bars + 16), sempty0 = smem_u32(bars + 32);     // [NS] TMEM slots
  const uint32_t qfull0 = smem_u32(bars + 48), qempty0 = smem_u32(bars + 50);     // [2]
  const uint32_t xchg0 = smem_u32(bars + 52);                                      // [4]

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint32_t rank_u = 0;
  if (C > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank_u));
  const int rank = (int)rank_u;
  const int cluster_id = blockIdx.x / C;
  const int nclusters = gridDim.x / C;
  const int units = c.R * c.L * c.h_kv;

  if (threadIdx.x == 0) {
    // full: the gather threads' cp.async arrivals, or (ktma) the feeder's one expect_tx arrival + TMA bytes
    const int fcount = ktma ? 1 : kRLoadWarps * 32;
    for (int s = 0; s < K::ST; ++s) { mbar_init(full0 + 8 * s, fcount); mbar_init(empty0 + 8 * s, 1); }
    for (int s = 0; s < K::NS; ++s) { mbar_init(sfull0 + 8 * s, 1); mbar_init(sempty0 + 8 * s, kREpiWarps / 2); }
    for (int b = 0; b < 2; ++b) { mbar_init(qfull0 + 8 * b, 1); mbar_init(qempty0 + 8 * b, 1); }
    for (int b = 0; b < 4; ++b) mbar_init(xchg0 + 8 * b, 1);   // [group][unit parity]: expect_tx + C senders' bytes
    int* of = reinterpret_cast<int*>(smem + K::OFF_F) + 12 * K::GW + 2 * 2 * C * K::GW * 2 + 8 * K::GW;
    of[0] = of[1] = -1;                                          // epilogue overflow flags (unit-tagged)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_q)));
  if (warp == 3 && lane == 0 && ktma) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_k)));
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (C > 1) cluster_sync_all();        // peers' barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const float scale = kLog2e * rsqrtf((float)D);

  struct UnitInfo { int r, l, h, T, slot, tb, nt; };
  auto unit_info = [&](int unit) {
    UnitInfo u;
    u.h = unit % c.h_kv;
    u.l = (unit / c.h_kv) % c.L;
    u.r = unit / (c.h_kv * c.L);
    u.T = c.seq_lens[u.r];
    u.slot = c.q_slots[u.r];
    const int ntot = (u.T + kTile - 1) / kTile;
    const int sr = (c.debug & 2u) ? C - 1 - rank : rank;      // tuning: reversed slice order (A/B)
    u.tb = (int)((long long)ntot * sr / C);
    u.nt = (int)((long long)ntot * (sr + 1) / C) - u.tb;       // <= NS (host sized C)
    return u;
  };

  if (warp < kREpi0 || warp >= kRLoad0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRProdRegs));
    if (warp == 0) {
      // ================= Q producer: the unit's G heads x w rows, one TMA box per 64-element slab
      if (lane == 0) {
        const uint64_t drop = policy_evict_first();
        for (int it = 0, unit = cluster_id; unit < units; ++it, unit += nclusters) {
          const UnitInfo u = unit_info(unit);
          const int qb = it & 1;
          mbar_wait_backoff(qempty0 + 8 * qb, ((it >> 1) & 1) ^ 1, 500);
          mbar_expect_tx(qfull0 + 8 * qb, K::Q_BYTES);
          const uint32_t qdst = smem_u32(smem + K::OFF_Q + qb * K::Q_BYTES);
          const int qrow = (u.l * c.M + u.slot) * W;
          for (int sl = 0; sl < K::SLABS; ++sl)
            tma_load_3d(qdst + sl * K::SLAB_Q, &tmap_q, sl * 64, u.h * G, qrow, qfull0 + 8 * qb, drop);
        }
      }
      __syncwarp();
    } else if (warp >= kRLoad0 && !ktma) {
      // ================= K gather: this CTA's tiles of every unit, in order (rows through the block table;
      // ids from the feeder; 16-B cp.async straight into the SW128 K-major stage)
      constexpr int CPR = D / 8;
      constexpr int RPP = kRLoadWarps * 32 / CPR;
      static_assert(RPP % 8 == 0, "the per-thread SW128 swizzle term needs rows-per-pass % 8 == 0");
      const int et = threadIdx.x - kRLoad0 * 32;
      const int cr = et % CPR, rsub = et / CPR;
      const uint32_t chunk_off = (uint32_t)(cr >> 3) * K::SLAB_K;
      const uint16_t* Kg = reinterpret_cast<const uint16_t*>(c.k_cache);
      const uint32_t ids_base = smem_u32(ids);
      const bool b_pow2 = (c.b & (c.b - 1)) == 0;
      const int b_log2 = 31 - __clz(c.b);
      const uint32_t dst_thr = (uint32_t)rsub * 128u + (uint32_t)(((cr & 7) ^ (rsub & 7)) << 4) + chunk_off;
      const uint32_t hD = (uint32_t)c.h_kv * D;
      int step = 0;
      for (int unit = cluster_id; unit < units; unit += nclusters) {
        const UnitInfo u = unit_info(unit);
        const uint16_t* lbase = Kg + (size_t)u.l * c.N_total * c.b * hD + (size_t)u.h * D + cr * 8;
        for (int i = 0; i < u.nt; ++i, ++step) {
          const int st = step % K::ST;
          const int t0 = (u.tb + i) * kTile;
          const int j0 = b_pow2 ? (t0 >> b_log2) : t0 / c.b;
          const uint32_t dst0 = smem_u32(Ks + st * K::STAGE_BYTES) + dst_thr;
          named_bar(6, kRLoadWarps * 32 + 32);                // feeder: ids of this tile landed, stage free
          const uint32_t sid = ids_base + (uint32_t)(step % kIdSlots) * kMaxIds * 4;
          uint32_t off[kTile / RPP];
#pragma unroll
          for (int k = 0; k < kTile / RPP; ++k) {
            const int t = t0 + RPP * k + rsub;
            const int jr = b_pow2 ? (t >> b_log2) : t / c.b;
            const int blk = lds_s32(sid + 4u * (uint32_t)min(max(jr - j0, 0), kMaxIds - 1));
            ZPC_CHECK(t >= u.T || (blk >= 0 && blk < c.N_total && t - jr * c.b < c.b));
            off[k] = ((uint32_t)blk * (uint32_t)c.b + (uint32_t)(t - jr * c.b)) * hD;
          }
#pragma unroll
          for (int k = 0; k < kTile / RPP; ++k)
            if (t0 + RPP * k + rsub < u.T) cp_async16(dst0 + (uint32_t)(RPP * k * 128), lbase + off[k]);
          cp_async_arrive_noinc(full0 + 8 * st);
        }
      }
    } else if (warp == 3) {
      // ================= feeder: block ids of each tile (4-byte cp.async into an smem ring, kIdAhead tiles
      // ahead) and the stage's release by the MMA; one named barrier with the gatherers publishes both
      static_assert(kIdSlots >= kIdAhead + 2, "id ring too small for the lookahead");
      int l_unit = cluster_id, l_i = 0;
      UnitInfo l_u = l_unit < units ? unit_info(l_unit) : UnitInfo{};
      const uint32_t ids_base = smem_u32(ids);
      auto issue_ids = [&](int slot) {
        while (l_unit < units && l_i >= l_u.nt) {
          l_unit += nclusters;
          l_i = 0;
          if (l_unit < units) l_u = unit_info(l_unit);
        }
        if (l_unit < units) {
          const int t0 = (l_u.tb + l_i) * kTile;
          const int j0 = t0 / c.b;
          const int nb = (min(t0 + kTile, l_u.T) - 1) / c.b - j0 + 1;
          if (lane < nb)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ids_base + (uint32_t)(slot * kMaxIds + lane) * 4u),
                         "l"(c.tables + (size_t)l_u.r * c.table_stride + j0 + lane) : "memory");
          ++l_i;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      int total = 0;
      for (int unit = cluster_id; unit < units; unit += nclusters) total += unit_info(unit).nt;
      int p_unit = cluster_id, p_i = 0;          // TMA path: the tile being issued
      UnitInfo p_u = l_u;
      const uint64_t keep = policy_evict_first();
#pragma unroll 1
      for (int k = 0; k < kIdAhead; ++k) issue_ids(k);
      for (int g = 0; g < total; ++g) {
        issue_ids((g + kIdAhead) % kIdSlots);
        if (g >= K::ST) {
          if (lane == 0) mbar_wait(empty0 + 8 * (g % K::ST), ((g / K::ST) & 1) ^ 1);
          __syncwarp();
        }
        asm volatile("cp.async.wait_group %0;" ::"n"(kIdAhead) : "memory");
        if (ktma) {
          // b % 128 == 0: the tile is 128 consecutive slots of one block, one head: SLABS boxes of 64 elements
          // x 128 rows (row stride h_kv*d) land in the SW128 K-major stage (no per-row gather instructions)
          __syncwarp();
          if (lane == 0) {
            while (p_unit < units && p_i >= p_u.nt) {
              p_unit += nclusters;
              p_i = 0;
              if (p_unit < units) p_u = unit_info(p_unit);
            }
            const int st = g % K::ST;
            const int t0 = (p_u.tb + p_i) * kTile;
            const int blk = lds_s32(ids_base + (uint32_t)((g % kIdSlots) * kMaxIds) * 4u);
            ZPC_CHECK(blk >= 0 && blk < c.N_total);
            const int row = (p_u.l * c.N_total + blk) * c.b + (t0 % c.b);
            const uint32_t dst = smem_u32(Ks + st * K::STAGE_BYTES);
            mbar_expect_tx(full0 + 8 * st, K::STAGE_BYTES);
            for (int sl = 0; sl < K::SLABS; ++sl)
              tma_load_3d(dst + sl * K::SLAB_K, &tmap_k, sl * 64, p_u.h, row, full0 + 8 * st, keep);
            ++p_i;
          }
          __syncwarp();
        } else {
          named_bar(6, kRLoadWarps * 32 + 32);
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp == 1) {
      // ================= MMA issuer (converged warp, elected lane): one UMMA per tile into TMEM slot
      // (tile counter) % NS, once the epilogue released the slot's previous tile
      int kstep = 0;
      for (int it = 0, unit = cluster_id; unit < units; ++it, unit += nclusters) {
        const int nt = __shfl_sync(0xffffffffu, unit_info(unit).nt, 0);
        const int qb = it & 1;
        mbar_wait(qfull0 + 8 * qb, (it >> 1) & 1);
        const uint64_t qd0 = sw128_desc(smem_u32(smem + K::OFF_Q + qb * K::Q_BYTES));
        for (int i = 0; i < nt; ++i, ++kstep) {
          const int s = kstep % K::ST, sl = kstep % K::NS;
          if (lane == 0 && kstep < 1024) RTRACE(4 * kstep, gtimer());
          mbar_wait(sempty0 + 8 * sl, ((kstep / K::NS) & 1) ^ 1);
          if (lane == 0 && kstep < 1024) RTRACE(4 * kstep + 1, gtimer());
          mbar_wait(full0 + 8 * s, (kstep / K::ST) & 1);
          if (lane == 0 && kstep < 1024) RTRACE(4 * kstep + 2, gtimer());
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async data -> tensor core
          tc_fence_after();
          const uint64_t kd0 = sw128_desc(smem_u32(Ks + s * K::STAGE_BYTES));
#pragma unroll
          for (int k = 0; k < K::KSTEPS; ++k)
            umma_elect(tmem + sl * K::GW, kd0 + (((k >> 2) * K::SLAB_K + (k & 3) * 32) >> 4),
                       qd0 + (((k >> 2) * K::SLAB_Q + (k & 3) * 32) >> 4), idesc_bf16(kTile, K::GW), k > 0);
          umma_commit_elect(empty0 + 8 * s);    // K stage free once the MMA completes
          umma_commit_elect(sfull0 + 8 * sl);   // the tile's logits are in slot sl
        }
        umma_commit_elect(qempty0 + 8 * qb);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kREpiRegs));
    // ================= epilogue: two groups of 4 warps (one per TMEM lane quarter, i.e. 32 tokens of every
    // tile, all G*w columns) take alternate units, so one group's sweeps overlap the other's cluster
    // exchange and unit start. Group grp works on units it with (it & 1) == grp, exchange parity grp.
    constexpr int GW = K::GW;
    const int ew = warp - kREpi0;
    const int q = warp & 3, grp = ew >> 2;
    float* fb = reinterpret_cast<float*>(smem + K::OFF_F);
    float* red = fb + grp * 6 * GW;          // [4][GW] cross-quarter reduction
    float* wref = fb + 12 * GW + 2 * 2 * C * GW * 2 + grp * 4 * GW;   // [4][GW] per-warp references
    volatile int* oflag = reinterpret_cast<volatile int*>(fb + 12 * GW + 2 * 2 * C * GW * 2 + 8 * GW);   // [2]
    float* mloc = red + 4 * GW;              // [GW] CTA-local column max (log2 domain; reference of sweep B)
    float* L2s = mloc + GW;                  // [GW] merged log2 normaliser
    // xbuf[grp][k & 1][C][GW] (max, sum) pairs of the group's k-th unit, PUSHED by every rank of the cluster with
    // st.async (remote shared-memory stores that complete_tx the receiver's barrier xchg[grp][k & 1]: no
    // cluster-scope fence, which would wait for the sender's outstanding global stores). Two per group: a rank
    // sends the k-th unit's pairs only after its exchange of the (k-1)-th completed, i.e. after every receiver
    // finished reading the (k-2)-th's (each rank sends k-1 after merging k-2).
    float2* xb0 = reinterpret_cast<float2*>(fb + 12 * GW) + grp * 2 * C * GW;
    float* pmg = red;                        // CTA-local column max (log2) before sending (reuses red row 0..)
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const int bid = 1 + grp;                 // the group's named barrier (128 threads)
    // 32-column chunk h of tile kt_i (this warp's 32 tokens)
    auto ld32 = [&](int kt_i, int h, float* v) {
      const uint32_t a = lane_base + (uint32_t)((kt_i % K::NS) * GW + h * 32);
      TMEM_LD16(a, v, 0);
      TMEM_LD16(a + 16, v, 16);
    };
    // causal / length mask of token t for chunk h (column h*32 + j <-> window row (h*32 + j) / G):
    // valid iff t <= T - W + (h*32 + j) / G
    auto mask32 = [&](float* v, int h, int t, int T) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = (t > T - W + (h * 32 + j) / G) ? -INFINITY : v[j];
    };
    using H0 = std::integral_constant<int, 0>;
    using H1 = std::integral_constant<int, 1>;
    // one sweep over the unit's tiles, two 32-column chunks per tile, the next chunk's TMEM load in flight
    // while the current one is processed. wait_full: wait for each tile's MMA (first sweep); release: the
    // group's last read of each slot (last sweep).
    auto sweep = [&](const UnitInfo& u, int kt0, bool wait_full, bool release, auto&& on_chunk) {
      if (u.nt == 0) return;                 // a short unit can leave a rank without tiles (R34)
      float va[32], vb[32];
      if (wait_full) { mbar_wait(sfull0 + 8 * (kt0 % K::NS), (kt0 / K::NS) & 1); tc_fence_after(); }
      ld32(kt0, 0, va);
      tmem_wait_ld();
      for (int i = 0; i < u.nt; ++i) {
        ld32(kt0 + i, 1, vb);
        on_chunk(i, H0{}, va);
        tmem_wait_ld();
        if (release) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(sempty0 + 8 * ((kt0 + i) % K::NS));
        }
        if (i + 1 < u.nt) {
          if (wait_full) {
            mbar_wait(sfull0 + 8 * ((kt0 + i + 1) % K::NS), ((kt0 + i + 1) / K::NS) & 1);
            tc_fence_after();
          }
          ld32(kt0 + i + 1, 0, va);
        }
        on_chunk(i, H1{}, vb);
        tmem_wait_ld();
      }
    };
    static_assert(GW == 64, "two 32-column chunks per tile");
    int kt = 0;                              // tiles of all earlier units (slot ring position)
    for (int it = 0, unit = cluster_id; unit < units; ++it, unit += nclusters) {
      const UnitInfo u = unit_info(unit);
      if ((it & 1) != grp) { kt += u.nt; continue; }
      const bool tr = q == 0 && lane == 0 && it < 512;
      const int xp = (it >> 1) & 1;
      float2* xb = xb0 + xp * C * GW;
      const uint32_t xbar = xchg0 + 8 * (grp * 2 + xp);
      if (q == 0 && lane == 0) mbar_expect_tx(xbar, (uint32_t)(C * GW * 8));   // the phase's one arrival
      if (tr) RTRACE(4096 + 8 * it + 0, gtimer());
      auto need_mask = [&](int i) { return (u.tb + i) * kTile + kTile - 1 > u.T - W; };   // warp-uniform
      const int tq = q * 32 + lane;
      float acc[GW];
      float mpub[GW / 128 + 1];                 // this thread's columns: published max (log2 domain)
      float spub[GW / 128 + 1];                 //                         published sum
      // ---- common case, ONE sweep: per-column sum of 2^(x*s - ref_q) with ref_q = the logit of the warp's first
      //      token in the slice (lane 0, tile 0), so the sum is >= 1 and no max sweep is needed; the four
      //      quarters' (ref, sum) pairs are merged like the cluster's. A logit ~100 log2 units above ref_q
      //      (the sum leaves fp32 range) sends the whole unit to the exact two-sweep path below.
      float* wr = wref + q * GW;                // this warp's references (log2 domain; 0 for an all-masked column)
#pragma unroll
      for (int j = 0; j < GW; ++j) acc[j] = 0.f;
      sweep(u, kt, true, false, [&](int i, auto hc, float* v) {
        constexpr int h = decltype(hc)::value;
        if (need_mask(i)) mask32(v, h, (u.tb + i) * kTile + tq, u.T);
        if (i == 0) {
          if (lane == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) wr[h * 32 + j] = v[j] > -INFINITY ? v[j] * scale : 0.f;
          }
          __syncwarp();
        }
        const float2* r2 = reinterpret_cast<const float2*>(wr + h * 32);   // (broadcast loads)
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 m2 = r2[j / 2];
          const uint64_t a2 = fma2(pk2(v[j], v[j + 1]), pk2(scale, scale), pk2(-m2.x, -m2.y));
          float a0, a1;
          upk2(a2, a0, a1);
          acc[h * 32 + j] += ex2f(a0);
          acc[h * 32 + j + 1] += ex2f(a1);
        }
      });
      bool ovf = false;
#pragma unroll
      for (int j = 0; j < GW; ++j) ovf |= !(acc[j] < 0x1p100f);
      if (__any_sync(0xffffffffu, ovf) && lane == 0) oflag[grp] = it + 1;   // unit-tagged: no reset needed
      warp_col_reduce<GW, false>(acc, lane);
#pragma unroll
      for (int k = 0; k < GW / 32; ++k) red[q * GW + reduced_col<GW>(lane, k)] = acc[k];
      named_bar(bid, 128);
      if (tr) RTRACE(4096 + 8 * it + 1, gtimer());
      if (oflag[grp] != it + 1) {
#pragma unroll
        for (int k = 0; k * 128 < GW; ++k) {
          const int col = q * 32 + lane + k * 128;
          if (col < GW) {
            float M = -INFINITY;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq)
              if (red[qq * GW + col] > 0.f) M = fmaxf(M, wref[qq * GW + col]);
            float S = 0.f;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq)
              if (red[qq * GW + col] > 0.f) S += red[qq * GW + col] * ex2f(wref[qq * GW + col] - M);
            mpub[k] = M;
            spub[k] = S;
          }
        }
      } else {
        // ---- exact path: sweep A (per-column max over this CTA's tokens), then sweep B against it
        named_bar(bid, 128);                    // everyone has read red before it is rewritten
#pragma unroll
        for (int j = 0; j < GW; ++j) acc[j] = -INFINITY;
        sweep(u, kt, false, false, [&](int i, auto hc, float* v) {
          constexpr int h = decltype(hc)::value;
          if (need_mask(i)) mask32(v, h, (u.tb + i) * kTile + tq, u.T);
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[h * 32 + j] = fmaxf(acc[h * 32 + j], v[j]);
        });
        warp_col_reduce<GW, true>(acc, lane);
#pragma unroll
        for (int k = 0; k < GW / 32; ++k) red[q * GW + reduced_col<GW>(lane, k)] = acc[k];
        named_bar(bid, 128);
#pragma unroll
        for (int k = 0; k * 128 < GW; ++k) {
          const int col = q * 32 + lane + k * 128;
          if (col < GW) {
            const float m = fmaxf(fmaxf(red[col], red[GW + col]), fmaxf(red[2 * GW + col], red[3 * GW + col]));
            mloc[col] = m > -INFINITY ? m * scale : 0.f;        // all masked here -> any finite reference
            mpub[k] = m > -INFINITY ? m * scale : -INFINITY;
          }
        }
        named_bar(bid, 128);
#pragma unroll
        for (int j = 0; j < GW; ++j) acc[j] = 0.f;
        const float2* mr2 = reinterpret_cast<const float2*>(mloc);   // (broadcast loads)
        sweep(u, kt, false, false, [&](int i, auto hc, float* v) {
          constexpr int h = decltype(hc)::value;
          if (need_mask(i)) mask32(v, h, (u.tb + i) * kTile + tq, u.T);
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float2 m2 = mr2[(h * 32 + j) / 2];
            const uint64_t a2 = fma2(pk2(v[j], v[j + 1]), pk2(scale, scale), pk2(-m2.x, -m2.y));
            float a0, a1;
            upk2(a2, a0, a1);
            acc[h * 32 + j] += ex2f(a0);
            acc[h * 32 + j + 1] += ex2f(a1);
          }
        });
        warp_col_reduce<GW, false>(acc, lane);
#pragma unroll
        for (int k = 0; k < GW / 32; ++k) red[q * GW + reduced_col<GW>(lane, k)] = acc[k];
        named_bar(bid, 128);
#pragma unroll
        for (int k = 0; k * 128 < GW; ++k) {
          const int col = q * 32 + lane + k * 128;
          if (col < GW) spub[k] = (red[col] + red[GW + col]) + (red[2 * GW + col] + red[3 * GW + col]);
        }
      }
      // ---- exchange: each column's (max, sum) pushed to slot [rank][col] of every rank's xbuf
      if (tr) RTRACE(4096 + 8 * it + 2, gtimer());
#pragma unroll
      for (int k = 0; k * 128 < GW; ++k) {
        const int col = q * 32 + lane + k * 128;
        if (col < GW) {
          const uint32_t la = smem_u32(xb + rank * GW + col);
#pragma unroll
          for (int rr = 0; rr < C; ++rr) st_async_v2(la, xbar, rr, mpub[k], spub[k]);
        }
      }
      mbar_wait(xbar, (it >> 2) & 1);            // every rank's pairs landed (complete_tx)
      if (tr) RTRACE(4096 + 8 * it + 3, gtimer());
      // merge into L2 = log2 sum_t 2^(x*s)
      for (int col = q * 32 + lane; col < GW; col += 128) {
        float M = -INFINITY, mv[C], sv[C];
#pragma unroll
        for (int rr = 0; rr < C; ++rr) {
          const float2 v2 = xb[rr * GW + col];
          mv[rr] = v2.x;
          sv[rr] = v2.y;
          M = fmaxf(M, mv[rr]);
        }
        float S = 0.f;
#pragma unroll
        for (int rr = 0; rr < C; ++rr)
          if (mv[rr] > -INFINITY) S += sv[rr] * ex2f(mv[rr] - M);
        const float L2 = M + lg2f(S);
        L2s[col] = L2;
        if (rank == 0) c.ws.lse[(size_t)unit * GW + col] = L2;
      }
      named_bar(bid, 128);
      // ---- sweep C: S[t] = (1/w) sum_u 2^(max_g (x*s - L2)), this thread's token over the whole window
      const float2* l2 = reinterpret_cast<const float2*>(L2s);
      float s4[4];
      sweep(u, kt, false, true, [&](int i, auto hc, float* v) {
        constexpr int h = decltype(hc)::value;
        const int t = (u.tb + i) * kTile + tq;
        if (h == 0) { s4[0] = s4[1] = s4[2] = s4[3] = 0.f; }
        if (need_mask(i)) mask32(v, h, t, u.T);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 n2 = l2[(h * 32 + j) / 2];
          const uint64_t a2 = fma2(pk2(v[j], v[j + 1]), pk2(scale, scale), pk2(-n2.x, -n2.y));
          upk2(a2, v[j], v[j + 1]);
        }
#pragma unroll
        for (int uu = 0; uu < 32 / G; ++uu) s4[uu & 3] += ex2f(gmax<G>(v + uu * G));
        if (h == 1 && t < u.T)
          c.ws.scores[(size_t)unit * c.max_seq_len + t] = ((s4[0] + s4[1]) + (s4[2] + s4[3])) * (1.0f / W);
      });
      if (tr) RTRACE(4096 + 8 * it + 4, gtimer());
      kt += u.nt;
    }
  }
  // ---- teardown
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  if (C > 1) cluster_sync_all();   // no CTA leaves while a peer may still read its partials
}

template <int G, int W, int D, int C>
cudaError_t launch_res(const Call& c, cudaStream_t s) {
  using K = CfgR<G, W, D, C>;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tq;
  const cuuint32_t estr[3] = {1, 1, 1};
  const cuuint64_t qdim[3] = {(cuuint64_t)c.d, (cuuint64_t)c.h_q, (cuuint64_t)c.L * c.M * c.w};
  const cuuint64_t qstr[2] = {(cuuint64_t)c.d * 2, (cuuint64_t)c.h_q * c.d * 2};
  const cuuint32_t qbox[3] = {64, (cuuint32_t)G, (cuuint32_t)W};
  if (enc(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(c.q_cache), qdim, qstr, qbox, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  // K as [rows = L*N_total*b][h_kv][d]: one box = 128 consecutive slots x 64 elements of one head (SW128)
  CUtensorMap tk;
  memset(&tk, 0, sizeof(tk));
  int ktma = 0;
  if (c.b % kTile == 0) {
    const cuuint64_t kdim[3] = {(cuuint64_t)c.d, (cuuint64_t)c.h_kv, (cuuint64_t)c.L * c.N_total * c.b};
    const cuuint64_t kstr[2] = {(cuuint64_t)c.d * 2, (cuuint64_t)c.h_kv * c.d * 2};
    const cuuint32_t kbox[3] = {64, 1, (cuuint32_t)kTile};
    if (enc(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, c.k_cache, kdim, kstr, kbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
        CUDA_SUCCESS)
      ktma = 1;   // (a TMA slab 0 + cp.async slab 1 split measured no faster: 0.187 vs 0.184 ms)
  }
  Call cc = c;
#ifdef ZPC_TUNING
  if (const char* e = getenv("ZPC_RES_KTMA")) ktma = std::min(ktma, atoi(e));   // A/B: 0 cp.async, 1 TMA
  if (const char* e = getenv("ZPC_SCORE_DEBUG")) cc.debug = (uint32_t)strtoul(e, nullptr, 10);
#endif
  auto kern = k_score_res<G, W, D, C>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
  if (e != cudaSuccess) return e;
  const int units = c.R * c.L * c.h_kv;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kRThreads);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int dev = 0, sms = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  int max_clusters = sms / C;
  cfg.gridDim = dim3(C);
  int qn = 0;
  if (cudaOccupancyMaxActiveClusters(&qn, kern, &cfg) == cudaSuccess && qn > 0) max_clusters = std::min(max_clusters, qn);
  cudaGetLastError();
  cfg.gridDim = dim3((unsigned)(std::min(units, max_clusters) * C));
  return cudaLaunchKernelEx(&cfg, kern, cc, tq, tk, ktma);
}

template <int G, int W>
cudaError_t launch_res_g(const Call& c, cudaStream_t s, bool* used) {
  using K = CfgR<G, W, 128, 8>;   // (NS does not depend on C)
  // a unit's slice must fit a rank's slot ring: ceil(tiles / C) <= NS (with <= NS / 2 the two epilogue groups'
  // units are resident at once; above it the second unit's MMAs wait for slots, no deadlock: a unit's exchange
  // never waits on a later unit). Among the sizes that fit, the least work per cluster, counting a unit's fixed
  // cost (exchange, pipeline fill) as two tiles: (units per cluster) x (tiles of the busiest rank + 2).
  // Measured at T = 2304 (18 tiles), score ms for C = 4 / 6 / 8: 1 request 0.057 / 0.059 / 0.076, 4 requests
  // 0.180 / 0.184 / 0.255 -> C = 4 (all 148 SMs, 5 tiles per rank)
  const int npt = (c.max_seq_len + kTile - 1) / kTile;
  const int units = c.R * c.L * c.h_kv;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int best = 0;
  long long best_cost = 0;
  for (int cs : {4, 6, 8}) {
    const int per_rank = (npt + cs - 1) / cs;
    if (per_rank > K::NS) continue;
    const int ncl = std::max(1, std::min(units, sms / cs));
    const long long cost = (long long)((units + ncl - 1) / ncl) * (per_rank + 2);
    if (best == 0 || cost < best_cost) { best = cs; best_cost = cost; }
  }
#ifdef ZPC_TUNING
  if (const char* e = getenv("ZPC_RES_C")) best = atoi(e);   // A/B: cluster size 4 / 6 / 8
#endif
  *used = true;
  switch (best) {
    case 4: return launch_res<G, W, 128, 4>(c, s);
    case 6: return launch_res<G, W, 128, 6>(c, s);
    case 8: return launch_res<G, W, 128, 8>(c, s);
    default: break;
  }
  *used = false;
  return cudaSuccess;
}

}  // namespace

// Two-pass bf16 calls with w = 16, d = 128, G = 4 whose longest unit fits the cluster's TMEM twice over
// (T <= 8 CTAs x 256/(G*w) tiles x 128 tokens = 4096 tokens at G*w = 64) -- the paper's operating point
// (Qwen3-8B). Others fall through (k_score_tc).
bool score_res_applies(const Call& c) {
  if (c.dtype != ZPC_BF16 || c.lse_in != nullptr || c.w != 16 || c.d != 128 || (c.variant & ZPC_V_SCORE_SERIAL))
    return false;
  if (c.b < 5 || c.G != 4) return false;
  // the largest cluster (8) holds two units of ceil(T / 128) / 8 tiles each in the NS slots
  return (c.max_seq_len + kTile - 1) / kTile <= 8 * (CfgR<4, 16, 128, 8>::NS / 2);
}

cudaError_t launch_score_res(const Call& c, cudaStream_t s, bool* used) {
  *used = false;
  if (!score_res_applies(c)) return cudaSuccess;
  if (c.R * c.L * c.h_kv == 0) { *used = true; return cudaSuccess; }
  switch (c.G) {
    case 4: return launch_res_g<4, 16>(c, s, used);
    default: return cudaSuccess;
  }
}

}  // namespace zpc
