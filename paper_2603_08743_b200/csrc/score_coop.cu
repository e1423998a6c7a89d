// a1 + a2 on 5th-generation tensor cores: the cooperative CTA-pair scoring kernel (default for
// two-pass bf16 calls with w = 32 and G in {5, 7, 8}).
//
// What it computes (Alg. 1 + §C.2): for one unit (request r, layer l, KV head h)
//   x[c,t] = q_c . k_t / sqrt(d)   for the G*w window columns c = u*G + g and tokens t < T,
//   LSE[c] = log sum_{t <= T-w+u} exp x[c,t]                          (softmax normaliser, pass 1)
//   S[t]   = (1/w) sum_{u: t <= T-w+u} exp(max_g (x[(u,g),t] - LSE[(u,g)]))        (pass 2)
//
// Why this design ("k_score_coop"): the two passes read every K tile twice. When a
// unit is scored by one SM, the second read comes a whole unit later and misses L2 (round 1: 1.84x the
// K bytes from DRAM). Here a unit's tokens are cut into CHUNKS of kt pair-tiles (256 tokens) that
// different CTA pairs score at the same time; each chunk publishes a partial log2-sum-exp per column to
// global memory, and a pair starts pass 2 of its chunk once every chunk of the unit has published. The
// second read of a tile then comes ~one chunk (~38-76 MB of traffic GPU-wide) after the first: an L2 hit.
//
//  * Work list: rounds of whole units packed onto the grid's pairs (k_coop_plan, one thread, request
//    order); pair p takes slot p of every round. Pass 2 of a round-rho chunk waits only for pass-1 work of
//    round-rho chunks, and a pair's pass-1 steps only wait for its own earlier steps, so no cycle exists
//    across pairs (DESIGN.md §6 gives the argument).
//  * Per pair: tcgen05.mma.cta_group::2. Each CTA holds the Q rows of half the window (its G*w/2 columns,
//    3 buffers) and 128 tokens of every 256-token pair-tile (4-stage K ring). Pass 1: M = 256 columns
//    (A = Q halves), N = 128 tokens per sub-step (64 K rows from each CTA) into two double-buffered TMEM
//    accumulators; pass 2: M = 256 tokens (A = K halves), N = G*w (B = Q halves) + a 9th K-step that
//    subtracts the normaliser (A_aug = ones, B_aug = bf16 split of -L2/s), so the accumulator already
//    holds q.k - L2/s.
//  * One merged step sequence (pass-1 tiles of chunk j interleaved with pass-2 tiles of an earlier
//    chunk) drives the K gather, the feeder, the stage relay and the MMA; a greedy rule keeps pass 2 of a
//    chunk >= delta steps behind its pass 1 (time for the cross-pair exchange) and pass 1 of chunk j
//    behind pass 2 of chunk j-3 (the Q buffer it reuses).
// Warp roles (768 threads, both CTAs): 0 Q producer (TMA), 1 MMA issuer (rank 0) / stage relay (rank 1),
// 2 combiner (chunk partials -> LSE -> B_aug), 3 feeder (block ids, stage release), 4-7 K gather
// (cp.async into SW128), 8-15 pass-1 epilogue (per-column online max/sum), 16-23 pass-2 epilogue.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <cuda_bf16.h>

#include "internal.h"
#include "tc_util.h"

namespace zpc {
namespace {

constexpr int kCLoadWarps = 4;
constexpr int kCEpi0 = 8;          // warps 0-7 producers, 8-23 pass-1 epilogue, 24-27 pass-2 epilogue
constexpr int kCP1Warps = 16;
constexpr int kCP2Warps = 4;
constexpr int kCThreads = (kCEpi0 + kCP1Warps + kCP2Warps) * 32;   // 896: 72 registers per thread at launch
constexpr int kCProdRegs = 48;
constexpr int kCP1Regs = 80;
constexpr int kCP2Regs = 72;   // launch allocation (no setmaxnreg)
static_assert(8 * kCProdRegs + kCP1Warps * kCP1Regs + kCP2Warps * kCP2Regs <= 2048, "register file: 65536 = 32 lanes x 2048");
#ifndef ZPC_COOP_POLY
#define ZPC_COOP_POLY 0   // eighths of the pass-1 exp2 pairs computed on the FMA pipe instead of MUFU
#endif
#ifndef ZPC_COOP_DELTA
#define ZPC_COOP_DELTA 12 // merged steps between a chunk's last pass-1 step and its first pass-2 step
#endif
#ifndef ZPC_COOP_KT
// pair-tiles per chunk (>= kCoopChunkTiles). Measured (production builds, one B200, score ms for kt = 16 / 32 /
// 64): qwen7b 7.69 / 7.48 / 7.47, qwen32b 34.2 / 33.3 / 32.5, prefix 23.3 / 22.4 / 22.0 (128 and 512 within noise
// of 64); qwen7b at kt = 4 / 8 / 16 / 64 on one box: 9.26 / 8.83 / 8.32 / 7.96 (delta 4 / 24 at kt = 8: 8.88 /
// 8.62): whole units per pair beat splitting a unit across pairs (the shorter pass-1 -> pass-2 distance does not
// buy L2 hits), so chunks only split units past 16K tokens.
#define ZPC_COOP_KT 64
#endif
#ifndef ZPC_COOP_HINTS
#define ZPC_COOP_HINTS 0  // CoopArgs::hints
#endif
constexpr int kQBufs = 3;
constexpr int kDescRing = 16;     // step descriptors in flight (feeder -> loaders, relay, MMA)
constexpr uint32_t kDescEnd = 0xFFFFFFFFu;
// step descriptor: bit 0 kind (0 pass 1, 1 pass 2), bit 1 first tile of the chunk, bit 2 last tile,
// bits 3..14 tile index k in the chunk, bits 15..30 chunk sequence number j of this pair
// (bits 1/2 follow the step's position in the chunk's sequence; the tile index is the tile it reads)
__device__ __forceinline__ uint32_t desc_pack(int kind, int k, int nt, int j, int tile) {
  return (uint32_t)kind | ((k == 0) ? 2u : 0u) | ((k + 1 == nt) ? 4u : 0u) | ((uint32_t)(tile & 0xFFF) << 3) |
         ((uint32_t)(j & 0xFFFF) << 15);
}
#ifndef ZPC_COOP_REV
#define ZPC_COOP_REV 0   // 1: pass 2 walks a chunk's tiles last-to-first: the tiles pass 1 read last are re-read first
                         // (measured: no fewer DRAM bytes, 2% slower -- the re-reads miss L2 either way)
#endif
// tile read by the k-th pass-2 step of a chunk of nt tiles
__device__ __forceinline__ int p2_tile(int k, int nt) { return ZPC_COOP_REV ? nt - 1 - k : k; }

// ------------------------------------------------------------------ pass-1 exp sums (packed)
template <int PE>
__host__ __device__ constexpr bool coop_poly_pair(int j) { return PE != 0 && (j & 7) >= 8 - PE; }
template <int N, int PE>
__device__ __forceinline__ float coop_sum_exp(const float* v, float scale, float m) {
  uint64_t acc[4] = {0, 0, 0, 0};
  const uint64_t S2 = pk2(scale, scale), NM2 = pk2(-m, -m);
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const uint64_t arg = fma2(pk2(v[2 * j], v[2 * j + 1]), S2, NM2);
    if (coop_poly_pair<PE>(j)) {
      // arguments are relative to a fixed reference and may be > 0: clamp at 126 so a huge logit gives
      // 2^126 (caught by the caller's 2^100 check) instead of a wrapped exponent
      float a0, a1;
      upk2(arg, a0, a1);
      acc[j & 3] = add2(acc[j & 3], ex2_poly4x2(pk2(fminf(a0, 126.f), fminf(a1, 126.f))));
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

// ------------------------------------------------------------------ work list
struct CoopArgs {
  int kt;          // pair-tiles (256 tokens) per chunk in this call
  int cmax;        // chunk stride of `part` per unit
  int delta;       // merged-step gap between a chunk's pass 1 and its pass 2
  int npairs;      // CTA pairs in the grid (slots per round)
  uint32_t* trace; // ZPC_TUNING builds: event timeline of pair 0, rank 0 (clock64 low words), else NULL
  int debug;       // ZPC_TUNING bisection: 1 no pass-1 math, 2 no pass-2 math, 4 no K gather, 8 no MMA
  int hints;       // bit 2: Q reads evict_first (else evict_last). (An L2::cache_hint operand on the K
                   // cp.async faults with an illegal instruction on this toolchain: measured, not used.)
  float* part;     // [units][cmax][G*w] partial log2-sum-exp of each chunk (log2 domain, scaled logits)
  int* cnt;        // [units][2] chunks of the unit published, per CTA rank (column half)
  int* rs;         // [units + 2] first work index of each round; rs[nr] = units; rs[units + 1] = nr
  int ktma;        // K tiles by TMA (b a power of two in 16..256), else the cp.async gather
  int lh_major;    // work order: 0 unit order (request-major); 1 (layer, head)-major, requests inner (shared
                   // prefix calls: the same (l, h) of many requests run at once, so their common prefix tiles
                   // are read from DRAM about once and from L2 by the others -- the prefix dedup)
};

// work index v -> unit (r*L + l)*h_kv + h
__device__ __forceinline__ int coop_unit(const Call& c, const CoopArgs& a, int v) {
  if (!a.lh_major) return v;
  const int lh = v / c.R, r = v - lh * c.R;
  return r * c.L * c.h_kv + lh;   // lh = l*h_kv + h
}

struct Chunk { int unit, ci, c, tb, nt, T, r, l, h, slot; };

// slot p of round rho -> chunk (false: the slot is empty in this round)
__device__ __forceinline__ bool coop_chunk(const Call& c, const CoopArgs& a, int rho, int p, Chunk& o) {
  const int HU = c.L * c.h_kv;
  int v = a.rs[rho], off = 0;
  const int v1 = a.rs[rho + 1];
  while (v < v1) {
    const int unit0 = coop_unit(c, a, v);
    const int r = unit0 / HU;
    const int T = c.seq_lens[r];
    const int npt = (T + 255) >> 8;
    const int cr = (npt + a.kt - 1) / a.kt;
    // a run of consecutive work items with the same chunk count: all of request r's units (unit order), or
    // one item ((l, h)-major order: consecutive items are different requests)
    const int nu = a.lh_major ? 1 : min(v1, (r + 1) * HU) - v;
    if (p < off + nu * cr) {
      const int q = p - off;
      o.unit = coop_unit(c, a, v + q / cr);
      o.ci = q % cr;
      o.c = cr;
      o.T = T;
      o.r = r;
      o.tb = (int)((long long)o.ci * npt / cr);
      o.nt = (int)((long long)(o.ci + 1) * npt / cr) - o.tb;
      o.h = o.unit % c.h_kv;
      o.l = (o.unit / c.h_kv) % c.L;
      o.slot = c.q_slots[r];
      return true;
    }
    off += nu * cr;
    v += nu;
  }
  return false;
}
struct ChunkIt { int rho, nr; };
__device__ __forceinline__ bool next_chunk(const Call& c, const CoopArgs& a, ChunkIt& it, int p, Chunk& o) {
  while (it.rho < it.nr) {
    const int rho = it.rho++;
    if (coop_chunk(c, a, rho, p, o)) return true;
  }
  return false;
}

// The merged step sequence, walked by the feeder alone (it publishes one descriptor per step): a step is
// one pair-tile of pass 1 of chunk j1 or of pass 2 of chunk j2 < j1. Greedy: alternate when both are
// allowed; pass 1 of chunk j needs pass 2 of chunk j-3 finished (its Q buffer); pass 2 of chunk j needs
// pass 1 of chunk j finished (hard) and `delta` steps since (soft: time for the other pairs' partials and
// the combine). State is scalar (registers); per-chunk data live in the shared chunk table.
struct Sched {
  int rho, nr, nch, j1, k1, j2, k2, step, last;
  bool exhausted;
  int kind, j, k, idx;   // the current step
};
// chunk table entry fields (ints): 0 T, 1 r, 2 l, 3 h, 4 tb, 5 unit (-1: end), 6 ci, 7 c, 8 nt, 9 slot,
// 10 end step of the chunk's pass 1 (feeder-private)
constexpr int kCtabInts = 16;

// ------------------------------------------------------------------ shared-memory layout
template <int G, int W, int D>
struct CfgC {
  static constexpr int GW = G * W;
  static constexpr int GWH = GW / 2;                   // columns per CTA (its half of the window rows)
  static constexpr int W2 = W / 2;
  static constexpr int SLABS = D / 64;                 // 64-element (128 B) K-chunks
  static constexpr int KSTEPS = D / 16;
  static constexpr int HALF = GWH / 2;                 // pass-2 B rows per CTA per column half (W/4 window rows)
  
  static constexpr uint32_t SLAB_Q = GWH * 128;        // GWH rows of 128 B; the pass-1 A operand reads 128
  static constexpr uint32_t Q_BYTES = SLAB_Q * SLABS;  // rows from a slab start (rows >= GWH: don't care)
  static constexpr uint32_t Q_TX = Q_BYTES;
  static constexpr uint32_t SLAB_K = 128 * 128;
  static constexpr uint32_t STAGE_BYTES = 128 * D * 2;
  static constexpr uint32_t AUG_A_BYTES = 128 * 32;
  static constexpr uint32_t AUG_B_BYTES = GWH * 32;    // per buffer (2 buffers)
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_AUG_A = kQBufs * Q_BYTES;
  static constexpr uint32_t OFF_AUG_B = OFF_AUG_A + AUG_A_BYTES;
  static constexpr uint32_t AUG_END = (OFF_AUG_B + 2 * AUG_B_BYTES + 1023) / 1024 * 1024;
  static constexpr uint32_t F_BYTES = (2 * 128 + 2 * 128) * 4;   // pm/ps[2][128] (token-slice merge)
  static constexpr uint32_t IDS_BYTES = kIdSlots * kMaxIds * 4;
  static constexpr uint32_t BAR_BYTES = 48 * 8;
  static constexpr uint32_t SCHED_BYTES = kDescRing * 4 + 8 * kCtabInts * 4;   // step descriptors + chunk table
  static constexpr uint32_t MISC = F_BYTES + IDS_BYTES + BAR_BYTES + SCHED_BYTES;
  static constexpr int STAGES_FIT = (int)((227 * 1024 - MISC - AUG_END) / STAGE_BYTES);
  static constexpr int ST = STAGES_FIT > 4 ? 4 : STAGES_FIT;
  static constexpr uint32_t OFF_K = AUG_END;
  static constexpr uint32_t OFF_F = OFF_K + ST * STAGE_BYTES;
  static constexpr uint32_t OFF_IDS = OFF_F + F_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_IDS + IDS_BYTES;
  static constexpr uint32_t OFF_SCHED = OFF_BAR + BAR_BYTES;
  static constexpr uint32_t SMEM = OFF_SCHED + SCHED_BYTES;   // the dynamic base is 1024-B aligned (checked)
  static_assert(GWH % 16 == 0 && GWH <= 128 && GWH > 64, "a CTA's columns: 8-row groups per half, <= 128 TMEM lanes");
  static_assert(W % 2 == 0 && (W == 32 || W == 16), "epilogue batching assumes w = 32 or 16");
  static_assert(ST >= 2 && ST <= 8, "K ring depth");
  static_assert(SMEM <= 227 * 1024, "dynamic shared memory per CTA");
  static_assert(SLAB_Q % 1024 == 0, "Q slabs must stay 1024-B aligned for SW128");
};

// event timeline (tuning builds): [0, 4*8192) MMA steps (t_top, t_full, t_ready, t_done), then
// [32768, +4*2048) combiner chunks (t_start, t_count, t_aug, unit), then [40960, +2*2048) pass-1 publish
#ifdef ZPC_TUNING
#define CDEBUG(bit) (a.debug & (bit))
#define CTRACE(i, v) do { if (a.trace && blockIdx.x == 0 && (i) < 49152) a.trace[(i)] = (uint32_t)(v); } while (0)
#else
#define CDEBUG(bit) false
#define CTRACE(i, v) do { } while (0)
#endif
__device__ __forceinline__ uint32_t clk32() { return (uint32_t)clock64(); }
__device__ __forceinline__ float ld_cg_f32(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------------ plan kernel
// Rounds of whole units, packed greedily in unit order onto `npairs` slots; each unit of request r has
// c_r = ceil(ceil(T_r/256) / kt) chunks. Also zeroes the arrival counters.
constexpr int kPlanStageR = 8192;   // requests whose chunk counts are staged in shared memory first
__global__ void __launch_bounds__(1024) k_coop_plan(Call c, CoopArgs a) {
  if (*c.status != ZPC_OK) return;
  __shared__ int crs[kPlanStageR];    // chunk count per request (the serial packing loop reads no global memory)
  const int HU = c.L * c.h_kv, units = c.R * HU;
  for (int i = threadIdx.x; i < 2 * units; i += blockDim.x) a.cnt[i] = 0;
  const bool staged = c.R <= kPlanStageR;
  if (staged)
    for (int r = threadIdx.x; r < c.R; r += blockDim.x) crs[r] = max(((c.seq_lens[r] + 255) / 256 + a.kt - 1) / a.kt, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int rho = 0, used = 0;
    a.rs[0] = 0;
    // runs of work items with one chunk count: per request (unit order) or per item ((l, h)-major)
    const int nruns = a.lh_major ? units : c.R;
    for (int run = 0; run < nruns; ++run) {
      const int r = a.lh_major ? run % c.R : run;
      const int cr = staged ? crs[r] : max(((c.seq_lens[r] + 255) / 256 + a.kt - 1) / a.kt, 1);
      if (cr > a.npairs) { *c.status = ZPC_ERR_SEQ_TOO_LONG; return; }   // host sized kt from max_seq_len
      int u = a.lh_major ? run : r * HU, m = a.lh_major ? 1 : HU;
      while (m > 0) {
        const int fit = (a.npairs - used) / cr;
        if (fit == 0) { a.rs[++rho] = u; used = 0; continue; }
        const int take = min(fit, m);
        used += take * cr;
        u += take;
        m -= take;
      }
    }
    a.rs[rho + 1] = units;
    a.rs[units + 1] = units > 0 ? rho + 1 : 0;
  }
}

// ------------------------------------------------------------------ the kernel
template <int G, int W, int D>
__global__ void __launch_bounds__(kCThreads, 1) k_score_coop(Call c, CoopArgs a, const __grid_constant__ CUtensorMap tmap_q,
                                                             const __grid_constant__ CUtensorMap tmap_k) {
  using K = CfgC<G, W, D>;
  if (*c.status != ZPC_OK) return;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();   // SW128 operands need the 1024-B aligned base
  uint8_t* Ks = smem + K::OFF_K;
  float* pm = reinterpret_cast<float*>(smem + K::OFF_F);   // [2][128] token-slice partial max (chunk-end merge)
  float* ps = pm + 256;                                     // [2][128] partial sums
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + K::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 46);
  int* ids = reinterpret_cast<int*>(smem + K::OFF_IDS);
  volatile uint32_t* desc = reinterpret_cast<volatile uint32_t*>(smem + K::OFF_SCHED);   // [kDescRing]
  // chunk table [8][16], written by the feeder when it fetches chunk j (entry j & 7, then ctab_full[j & 7]):
  // T, r, l, h, tb, unit (-1: no more chunks), ci, c, nt, slot
  volatile int* ctab = reinterpret_cast<volatile int*>(smem + K::OFF_SCHED + kDescRing * 4);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + 8);
  const uint32_t accf0 = smem_u32(bars + 16), acce0 = smem_u32(bars + 20);   // 0, 1: pass-1 buffers, 2, 3: pass-2 halves
  const uint32_t qfull0 = smem_u32(bars + 24), qempty0 = smem_u32(bars + 27);
  const uint32_t augf0 = smem_u32(bars + 30), auge0 = smem_u32(bars + 32);
  const uint32_t p1pub0 = smem_u32(bars + 34);     // [4] pass-1 partials of chunk j stored (-> combiner)
  const uint32_t ctabf0 = smem_u32(bars + 38);     // [8] chunk table entry j & 7 written

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint32_t rank_u;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank_u));
  const int rank = (int)rank_u;
  const int pair = blockIdx.x / 2;
  const int units = c.R * c.L * c.h_kv;
  const int nr = a.rs[units + 1];

  if (threadIdx.x == 0) {
    for (int s = 0; s < K::ST; ++s) {
      // the gather threads' cp.async arrivals, or (a.ktma) the feeder's one expect_tx arrival; + rank 1's relay
      mbar_init(full0 + 8 * s, (a.ktma ? 1 : kCLoadWarps * 32) + (rank == 0 ? 1 : 0));
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int i = 0; i < 4; ++i) { mbar_init(accf0 + 8 * i, 1); mbar_init(acce0 + 8 * i, i < 2 ? kCP1Warps : 2 * kCP2Warps); }
    for (int b = 0; b < kQBufs; ++b) { mbar_init(qfull0 + 8 * b, rank == 0 ? 2 : 1); mbar_init(qempty0 + 8 * b, 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(augf0 + 8 * b, 2); mbar_init(auge0 + 8 * b, 1); }
    for (int b = 0; b < 4; ++b) mbar_init(p1pub0 + 8 * b, 1);
    for (int b = 0; b < 8; ++b) mbar_init(ctabf0 + 8 * b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_q)));
  {
    // A_aug rows: bf16 1.0 in k = 0..2; both B_aug buffers start all zero (k = 3..15 stay 0)
    uint4* aug = reinterpret_cast<uint4*>(smem + K::OFF_AUG_A);
    for (int i = threadIdx.x; i < (int)((K::AUG_A_BYTES + 2 * K::AUG_B_BYTES) / 16); i += kCThreads) {
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (i < (int)(K::AUG_A_BYTES / 16) && ((i >> 3) & 1) == 0) v = make_uint4(0x3F803F80u, 0x00003F80u, 0u, 0u);
      aug[i] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const float scale = kLog2e * rsqrtf((float)D);

  if (warp < kCEpi0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCProdRegs));
    if (warp == 0) {
      // ================= Q producer: this CTA's half of the window of chunk j -> buffer j % 3
      if (lane == 0) {
        // Q of a unit is read by all its chunks' pairs at about the same time
        const uint64_t keep = (a.hints & 4) ? policy_evict_first() : policy_evict_last();
        for (int j = 0;; ++j) {
          mbar_wait_backoff(ctabf0 + 8 * (j & 7), (uint32_t)((j >> 3) & 1), 200);
          const volatile int* ce = ctab + kCtabInts * (j & 7);
          if (ce[5] < 0) break;
          const int l = ce[2], h = ce[3], slot = ce[9];
          const int qb = j % kQBufs;
          const uint32_t par = (uint32_t)((j / kQBufs) & 1);
          mbar_wait_backoff(qempty0 + 8 * qb, par ^ 1u, 200);
          mbar_expect_tx(qfull0 + 8 * qb, K::Q_TX);
          const uint32_t qdst = smem_u32(smem + K::OFF_Q + qb * K::Q_BYTES);
          const int qrow = (l * c.M + slot) * W + rank * K::W2;
          for (int sl = 0; sl < K::SLABS; ++sl)
            tma_load_3d(qdst + sl * K::SLAB_Q, &tmap_q, sl * 64, h * G, qrow, qfull0 + 8 * qb, keep);
          if (rank == 1) {   // relay: rank 0's MMA reads both halves
            mbar_wait_backoff(qfull0 + 8 * qb, par, 200);
            mbar_remote_arrive(qfull0 + 8 * qb, 0);
          }
        }
      }
      __syncwarp();
    } else if (warp == 1 && rank == 1) {
      // ================= rank 1: relay each landed K stage to rank 0's full barrier
      if (lane == 0) {
        for (int g = 0;; ++g) {
          mbar_wait(full0 + 8 * (g % K::ST), (g / K::ST) & 1);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_remote_arrive(full0 + 8 * (g % K::ST), 0);
          if (desc[g % kDescRing] == kDescEnd) break;
        }
      }
      __syncwarp();
    } else if (warp == 2) {
      // ================= combiner: publishes this CTA's pass-1 partials of chunk j (release add to the
      // unit's counter), waits for every chunk of the unit, combines them into the LSE of this CTA's
      // columns and writes it into B_aug[j & 1] as the bf16 split of -L2/s
      constexpr int CPL = (K::GWH + 31) / 32;
      constexpr int CQ = 8;   // chunk partials loaded per batch (all issued before the math)
      for (int j = 0;; ++j) {
        mbar_wait(ctabf0 + 8 * (j & 7), (uint32_t)((j >> 3) & 1));
        const volatile int* ce = ctab + kCtabInts * (j & 7);
        const int unit = ce[5], ci = ce[6], cc = ce[7];
        if (unit < 0) break;
        int* cp = a.cnt + (size_t)unit * 2 + rank;
        if (lane == 0) {
          if (j < 2048) { CTRACE(32768 + 4 * j, clk32()); CTRACE(32768 + 4 * j + 3, unit); }
          mbar_wait(p1pub0 + 8 * (j & 3), (uint32_t)((j >> 2) & 1));   // this CTA's partials are stored
          // release at gpu scope: cumulative over the pass-1 warps' partial stores this lane acquired
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cp) : "memory");
          long long spins = 0;
          unsigned long long t0 = 0;
          while (ld_acquire_s32(cp) < cc) {
            __nanosleep(64);
            if (spins++ == 0) t0 = gtime_ns();
            else if ((spins & 63) == 0 && gtime_ns() - t0 > kWaitLimitNs) {   // never hang silently
#ifdef ZPC_DEBUG_WAITS
              printf("zpc coop counter timeout: block %d unit %d have %d need %d\n", blockIdx.x, unit, ld_acquire_s32(cp), cc);
#endif
              __trap();
            }
          }
          if (j < 2048) CTRACE(32768 + 4 * j + 1, clk32());
        }
        __syncwarp();
        // every partial of the unit is published (lane 0's acquire, ordered to the warp by the syncwarp):
        // all loads are issued before any is used (entries beyond cc are clamped in range, then masked)
        const float* pp = a.part + ((size_t)unit * a.cmax) * K::GW + rank * K::GWH;
        float M[CPL], S[CPL];
#pragma unroll
        for (int i = 0; i < CPL; ++i) { M[i] = -INFINITY; S[i] = 0.f; }
        for (int q0 = 0; q0 < cc; q0 += CQ) {
          float v[CPL][CQ];
#pragma unroll
          for (int i = 0; i < CPL; ++i)
#pragma unroll
            for (int q = 0; q < CQ; ++q)
              v[i][q] = ld_cg_f32(pp + (size_t)min(q0 + q, a.cmax - 1) * K::GW + min(lane + 32 * i, K::GWH - 1));
#pragma unroll
          for (int i = 0; i < CPL; ++i)
#pragma unroll
            for (int q = 0; q < CQ; ++q) {
              const float x = (q0 + q < cc) ? v[i][q] : -INFINITY;
              const float Mn = fmaxf(M[i], x);
              if (Mn > -INFINITY) { S[i] = S[i] * ex2f(M[i] - Mn) + ex2f(x - Mn); M[i] = Mn; }
            }
        }
        const int ab = j & 1;
        mbar_wait(auge0 + 8 * ab, (uint32_t)(((j >> 1) & 1) ^ 1));   // pass-2 MMAs of chunk j-2 done
        uint8_t* augb = smem + K::OFF_AUG_B + ab * K::AUG_B_BYTES;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          const int col = lane + 32 * i;
          if (col < K::GWH) {
            const float L2 = M[i] + lg2f(S[i]);
            const float nv = -L2 / scale;
            const __nv_bfloat16 hi = __float2bfloat16_rn(nv);
            const float r1 = nv - __bfloat162float(hi);
            const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
            const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
            const uint32_t w0 = (uint32_t)__bfloat16_as_ushort(hi) | ((uint32_t)__bfloat16_as_ushort(mid) << 16);
            const uint32_t w1 = (uint32_t)__bfloat16_as_ushort(lo);
            *reinterpret_cast<uint2*>(augb + (col >> 3) * 256 + (col & 7) * 16) = make_uint2(w0, w1);
            if (ci == 0) c.ws.lse[(size_t)unit * K::GW + rank * K::GWH + col] = L2;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.acq_rel.cluster;" ::: "memory");
          mbar_remote_arrive(augf0 + 8 * ab, 0);
          if (j < 2048) CTRACE(32768 + 4 * j + 2, clk32());
        }
        __syncwarp();
      }
    } else if (warp >= 4 && warp < 4 + kCLoadWarps && !a.ktma) {
      // ================= K gather of this CTA's 128 tokens of the step's pair-tile (16-B cp.async, SW128)
      constexpr int CPR = D / 8;
      constexpr int RPP = kCLoadWarps * 32 / CPR;
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
      for (int g = 0;; ++g) {
        const int st = g % K::ST;
        named_bar(4, kCLoadWarps * 32 + 32);                     // feeder: descriptor + ids of step g, stage free
        const uint32_t dsc = desc[g % kDescRing];
        if (dsc == kDescEnd) { cp_async_arrive_noinc(full0 + 8 * st); break; }   // lets the MMA / relay see the end
        const int k = (dsc >> 3) & 0xFFF, j = (int)(dsc >> 15);
        const volatile int* ci = ctab + kCtabInts * (j & 7);            // T, r, l, h, tb
        const int T = ci[0], tb = ci[4];
        const int t0 = (tb + k) * 2 * kTile + rank * kTile;
        const int j0 = b_pow2 ? (t0 >> b_log2) : t0 / c.b;
        const uint16_t* lbase = Kg + (size_t)ci[2] * c.N_total * c.b * hD + (size_t)ci[3] * D + cr * 8;
        const uint32_t dst0 = smem_u32(Ks + st * K::STAGE_BYTES) + dst_thr;
        const uint32_t sid = ids_base + (uint32_t)(g % kIdSlots) * kMaxIds * 4;
        if (CDEBUG(4)) {
          // bisection: no K loads
        } else if (c.b == 16) {
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
          for (int kq = 0; kq < kTile / RPP; ++kq) {
            const int t = t0 + RPP * kq + rsub;
            const int jr = b_pow2 ? (t >> b_log2) : t / c.b;
            const int blk = lds_s32(sid + 4u * (uint32_t)min(max(jr - j0, 0), kMaxIds - 1));
            ZPC_CHECK(t >= T || (blk >= 0 && blk < c.N_total && t - jr * c.b < c.b));
            off[kq] = ((uint32_t)blk * (uint32_t)c.b + (uint32_t)(t - jr * c.b)) * hD;
          }
#pragma unroll
          for (int kq = 0; kq < kTile / RPP; ++kq)
            if (t0 + RPP * kq + rsub < T) cp_async16(dst0 + (uint32_t)(RPP * kq * 128), lbase + off[kq]);
        }
        cp_async_arrive_noinc(full0 + 8 * st);
      }
    } else if (warp == 3) {
      // ================= feeder: walks the merged schedule (the only role that does), kIdAhead steps ahead:
      // step descriptor + chunk table entry + the tile's block ids; then the stage release
      const uint64_t kpol = policy_evict_last();   // K tiles are re-read by pass 2
      Sched ls;
      ls.rho = 0; ls.nr = nr; ls.nch = ls.j1 = ls.k1 = ls.j2 = ls.k2 = ls.step = 0; ls.last = 1; ls.exhausted = false;
      const uint32_t ids_base = smem_u32(ids);
      bool ended = false;
      // fetch chunks up to j1 + 1 into the table (one ahead, so no table walk sits on a chunk boundary)
      auto fetch = [&]() {
        while (ls.nch <= ls.j1 + 1 && !ls.exhausted) {
          Chunk u;
          ChunkIt it{ls.rho, ls.nr};
          const bool got = next_chunk(c, a, it, pair, u);
          ls.rho = it.rho;
          volatile int* ce = ctab + kCtabInts * (ls.nch & 7);
          if (lane == 0) {
            if (got) {
              ce[0] = u.T; ce[1] = u.r; ce[2] = u.l; ce[3] = u.h; ce[4] = u.tb;
              ce[5] = u.unit; ce[6] = u.ci; ce[7] = u.c; ce[8] = u.nt; ce[9] = u.slot;
            } else {
              ce[5] = -1;
            }
            mbar_arrive(ctabf0 + 8 * (ls.nch & 7));
          }
          __syncwarp();
          if (got) ++ls.nch;
          else ls.exhausted = true;
        }
      };
      auto sched_next = [&]() -> bool {
        fetch();
        const bool p1ok = ls.j1 < ls.nch && ls.j2 > ls.j1 - kQBufs;
        const bool p2hard = ls.j2 < ls.j1;
        const bool p2soft = p2hard && ls.step - ctab[kCtabInts * (ls.j2 & 7) + 10] >= a.delta;
        int kind;
        if (p1ok && p2soft) kind = ls.last ^ 1;
        else if (p1ok) kind = 0;
        else if (p2hard) kind = 1;
        else return false;
        ls.idx = ls.step;
        ls.kind = kind;
        if (kind == 0) {
          ls.j = ls.j1;
          ls.k = ls.k1;
          if (++ls.k1 == ctab[kCtabInts * (ls.j1 & 7) + 8]) {
            ls.k1 = 0;
            if (lane == 0) ctab[kCtabInts * (ls.j1 & 7) + 10] = ls.step + 1;
            __syncwarp();
            ++ls.j1;
          }
        } else {
          ls.j = ls.j2;
          ls.k = ls.k2;
          if (++ls.k2 == ctab[kCtabInts * (ls.j2 & 7) + 8]) { ls.k2 = 0; ++ls.j2; }
        }
        ls.last = kind;
        ++ls.step;
        return true;
      };
      auto prepare = [&](int g) {   // step g -> descriptor slot g % kDescRing, id slot g % kIdSlots
        uint32_t dsc = kDescEnd;
        if (!ended && sched_next()) {
          const volatile int* ce = ctab + kCtabInts * (ls.j & 7);
          const int T = ce[0], r = ce[1], tb = ce[4], nt = ce[8];
          const int tile = ls.kind == 1 ? p2_tile(ls.k, nt) : ls.k;
          dsc = desc_pack(ls.kind, ls.k, nt, ls.j, tile);
          const int t0 = (tb + tile) * 2 * kTile + rank * kTile;
          if (t0 < T) {
            const int j0 = t0 / c.b;
            const int nb = (min(t0 + kTile, T) - 1) / c.b - j0 + 1;
            if (lane < nb)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ids_base + (uint32_t)((g % kIdSlots) * kMaxIds + lane) * 4u),
                           "l"(c.tables + (size_t)r * c.table_stride + j0 + lane) : "memory");
          }
        } else {
          ended = true;
        }
        if (lane == 0) desc[g % kDescRing] = dsc;
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      static_assert(kDescRing >= kIdAhead + 3 * 4 && kIdSlots >= kIdAhead + 2, "descriptor / id rings too small");
#pragma unroll 1
      for (int k = 0; k < kIdAhead; ++k) prepare(k);
      for (int g = 0;; ++g) {
        prepare(g + kIdAhead);
        if (g >= K::ST) {
          if (lane == 0) mbar_wait(empty0 + 8 * (g % K::ST), ((g / K::ST) & 1) ^ 1);
          __syncwarp();
        }
        asm volatile("cp.async.wait_group %0;" ::"n"(kIdAhead) : "memory");
        if (a.ktma) {
          // K by TMA (b a power of two in 16..256): one box of R = min(b, 128) consecutive slots x 64 elements
          // of head h per block the CTA's 128 tokens touch, per slab, straight into the SW128 K-major stage
          __syncwarp();
          const uint32_t dsc = desc[g % kDescRing];
          if (lane == 0) {
            const int st = g % K::ST;
            if (dsc == kDescEnd) {
              mbar_arrive(full0 + 8 * st);          // lets the MMA / relay see the end
            } else {
              const int k = (dsc >> 3) & 0xFFF, j = (int)(dsc >> 15);
              const volatile int* ce = ctab + kCtabInts * (j & 7);
              const int T = ce[0], l = ce[2], h = ce[3], tb = ce[4];
              const int t0 = (tb + k) * 2 * kTile + rank * kTile;
              const int R = min(c.b, kTile);
              const int nbox = t0 < T ? (min(t0 + kTile, T) - 1) / R - t0 / R + 1 : 0;
              mbar_expect_tx(full0 + 8 * st, (uint32_t)(nbox * K::SLABS * R * 128));
              const uint32_t sid = ids_base + (uint32_t)(g % kIdSlots) * kMaxIds * 4;
              const uint32_t dst0 = smem_u32(Ks + st * K::STAGE_BYTES);
              for (int x = 0; x < nbox; ++x) {
                const int tt = t0 + x * R;          // first token of box x
                const int blk = lds_s32(sid + 4u * (uint32_t)(tt / c.b - t0 / c.b));
                ZPC_CHECK(blk >= 0 && blk < c.N_total);
                const int row = (l * c.N_total + blk) * c.b + tt % c.b;
                for (int sl = 0; sl < K::SLABS; ++sl)
                  tma_load_3d(dst0 + sl * K::SLAB_K + (uint32_t)(x * R * 128), &tmap_k, sl * 64, h, row,
                              full0 + 8 * st, kpol);
              }
            }
          }
          __syncwarp();
          if (dsc == kDescEnd) break;
          continue;
        }
        named_bar(4, kCLoadWarps * 32 + 32);
        if (desc[g % kDescRing] == kDescEnd) break;
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp == 1 && rank == 0) {
      // ================= MMA issuer (rank 0 only; converged warp, elected lane issues); the step
      // descriptors come from the feeder (visible once the stage's full barrier completes)
      int n1 = 0, n2 = 0;
      const uint64_t aug_a = none_desc(smem_u32(smem + K::OFF_AUG_A), 128, 256);
      constexpr uint32_t kId1 = idesc_bf16(256, kTile), kId2 = idesc_bf16(256, K::GWH);
      if (lane == 0) { CTRACE(49148, clk32()); CTRACE(49149, (uint32_t)gtime_ns()); }
      for (int g = 0;; ++g) {
        const int st = g % K::ST;
        if (g < 8192 && lane == 0) CTRACE(4 * g, clk32());
        mbar_wait_cluster(full0 + 8 * st, (g / K::ST) & 1);
        const uint32_t dsc = desc[g % kDescRing];
        if (dsc == kDescEnd) break;
        if (g < 8192 && lane == 0) CTRACE(4 * g + 1, (clk32() & ~3u) | (dsc & 3u));
        const int kind = dsc & 1, j = (int)(dsc >> 15);
        const int qb = j % kQBufs;
        const uint64_t qd = sw128_desc(smem_u32(smem + K::OFF_Q + qb * K::Q_BYTES));
        const uint64_t kd0 = sw128_desc(smem_u32(Ks + st * K::STAGE_BYTES));
        if (kind == 0) {
          if (dsc & 2u) mbar_wait_cluster(qfull0 + 8 * qb, (uint32_t)((j / kQBufs) & 1));
          // pass 1: two sub-steps of N = 128 tokens (64 K rows from each CTA)
#pragma unroll 1
          for (int hs = 0; hs < 2; ++hs, ++n1) {
            const int ab = n1 & 1;
            mbar_wait_cluster(acce0 + 8 * ab, ((n1 >> 1) & 1) ^ 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < K::KSTEPS; ++kk)
              if (!CDEBUG(8)) umma2_elect(tmem + ab * 128, qd + (((kk >> 2) * K::SLAB_Q + (kk & 3) * 32) >> 4),
                          kd0 + (((kk >> 2) * K::SLAB_K + hs * 64 * 128 + (kk & 3) * 32) >> 4), kId1, kk > 0);
            umma2_commit_elect(accf0 + 8 * ab);
            if (hs == 0 && g < 8192 && lane == 0) CTRACE(4 * g + 2, clk32());
          }
        } else {
          // pass 2: two column halves (N = G*w/2: rows [h*HALF, +HALF) of each CTA's Q half and of B_aug),
          // each into its own TMEM buffer (columns 256 + h*GWH), so the epilogue drains one while the
          // tensor core fills the other
          const int ab = j & 1;
          if (dsc & 2u) mbar_wait_cluster(augf0 + 8 * ab, (uint32_t)((j >> 1) & 1));
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            mbar_wait_cluster(acce0 + 8 * (2 + h), (n2 & 1) ^ 1);
            if (h == 0 && g < 8192 && lane == 0) CTRACE(4 * g + 2, clk32());
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_fence_after();
            const uint64_t qdh = sw128_desc(smem_u32(smem + K::OFF_Q + qb * K::Q_BYTES) + h * K::HALF * 128);
            const uint64_t aug_b =
                none_desc(smem_u32(smem + K::OFF_AUG_B + ab * K::AUG_B_BYTES) + h * (K::HALF / 8) * 256, 128, 256);
            const uint32_t dacc = tmem + 256 + h * K::GWH;
#pragma unroll
            for (int kk = 0; kk < K::KSTEPS; ++kk)
              if (!CDEBUG(8)) umma2_elect(dacc, kd0 + (((kk >> 2) * K::SLAB_K + (kk & 3) * 32) >> 4),
                                          qdh + (((kk >> 2) * K::SLAB_Q + (kk & 3) * 32) >> 4), kId2, kk > 0);
            if (!CDEBUG(8)) umma2_elect(dacc, aug_a, aug_b, kId2, 1);
            umma2_commit_elect(accf0 + 8 * (2 + h));
          }
          ++n2;
          if (dsc & 4u) {
            umma2_commit_elect(auge0 + 8 * ab);        // B_aug[ab] free once this chunk's pass 2 is done
            umma2_commit_elect(qempty0 + 8 * qb);      // and the chunk's Q buffer
          }
        }
        umma2_commit_elect(empty0 + 8 * st);
        if (g < 8192 && lane == 0) CTRACE(4 * g + 3, clk32());
      }
      if (lane == 0) { CTRACE(49150, clk32()); CTRACE(49151, (uint32_t)gtime_ns()); }
    }
  } else if (warp < kCEpi0 + kCP1Warps) {
    // ================= pass-1 warps (16): lane quarter q = local columns q*32 + lane. Warp tq of a quarter
    // takes sub-step hs = tq >> 1 of every tile (buffer hs) and the 64 tokens of rank tq & 1 in it, so the
    // two warp pairs of a quarter alternate buffers: while one pair computes, the MMA refills the other.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kCP1Regs));
    const int q = warp & 3;
    const int tq = (warp - kCEpi0) >> 2;
    const int hs = tq >> 1;
    const int lc = q * 32 + lane;
    const bool col_ok = lc < K::GWH;
    const bool warp_cols = q * 32 < K::GWH;
    const int gcol = rank * K::GWH + lc;
    const int u1 = col_ok ? gcol / G : 0;
    const uint32_t tbase0 = tmem + ((uint32_t)(q * 32) << 16) + hs * 128 + (tq & 1) * 64;
    constexpr int NB = 64;
    int n1 = 0;   // tiles processed
    for (int jp = 0;; ++jp) {
      mbar_wait(ctabf0 + 8 * (jp & 7), (uint32_t)((jp >> 3) & 1));
      Chunk A;
      {
        const volatile int* ce = ctab + kCtabInts * (jp & 7);
        A.unit = ce[5];
        if (A.unit < 0) break;
        A.T = ce[0]; A.tb = ce[4]; A.ci = ce[6]; A.nt = ce[8];
      }
      const int limit1 = A.T - W + u1;
      // fixed reference per chunk (no per-batch max tree): m is set from the first batch with a valid
      // token; a batch whose sum leaves [0, 2^100) -- a logit ~100 log2 units above the reference -- is
      // redone against its own maximum (rescaling the running sum), so no exponent can overflow
      float m = -INFINITY, ssum = 0.f;
#pragma unroll 1
      for (int k = 0; k < A.nt; ++k, ++n1) {
        if (warp == kCEpi0 && lane == 0 && n1 < 1024) CTRACE(45056 + 4 * n1, clk32());
        mbar_wait_lean(accf0 + 8 * hs, (uint32_t)(n1 & 1));
        if (warp == kCEpi0 && lane == 0 && n1 < 1024) CTRACE(45056 + 4 * n1 + 1, clk32());
        tc_fence_after();
        // first token of this warp's 64: rank (tq & 1)'s K rows hs*64 .. of the pair-tile
        const int tb = (A.tb + k) * 2 * kTile + (tq & 1) * kTile + hs * 64;
        if (tb >= A.T || !warp_cols) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_remote_arrive_relaxed(acce0 + 8 * hs, 0);
          continue;
        }
        float vp[NB];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) TMEM_LD16(tbase0 + kk * 16, vp, kk * 16);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_remote_arrive_relaxed(acce0 + 8 * hs, 0);
        if (warp == kCEpi0 && lane == 0 && n1 < 1024) CTRACE(45056 + 4 * n1 + 2, clk32());
        if (tb + NB - 1 > A.T - W) {
#pragma unroll
          for (int jj = 0; jj < NB; ++jj) vp[jj] = (tb + jj > limit1) ? -INFINITY : vp[jj];
        }
        auto vmax = [&](const float* v) {
          float t3[21];
#pragma unroll
          for (int jj = 0; jj < 21; ++jj) t3[jj] = max3f(v[3 * jj], v[3 * jj + 1], v[3 * jj + 2]);
          float r = v[63];
#pragma unroll
          for (int jj = 0; jj < 21; jj += 3) r = fmaxf(r, max3f(t3[jj], t3[jj + 1], t3[jj + 2]));
          return r;
        };
        if (m == -INFINITY) m = vmax(vp) * scale;   // first batch of the chunk (or all masked so far)
        if (CDEBUG(1)) { ssum += vp[0]; continue; }
        if (m > -INFINITY) {
          float bsum = coop_sum_exp<NB, ZPC_COOP_POLY>(vp, scale, m);
          if (!(bsum < 0x1p100f)) {
            const float mn = fmaxf(m, vmax(vp) * scale);
            ssum *= ex2f(m - mn);
            m = mn;
            bsum = coop_sum_exp<NB, 0>(vp, scale, m);
          }
          ssum += bsum;
        }
        if (warp == kCEpi0 && lane == 0 && n1 < 1024) CTRACE(45056 + 4 * n1 + 3, __float_as_uint(ssum) == 1u ? 0u : clk32());
      }
      // ---- end of chunk A's pass 1: merge the four token slices (two rounds through smem) -> part
      auto merge = [&](float mo, float so) {
        const float mm = fmaxf(m, mo);
        const float mr = mm > -INFINITY ? mm : 0.f;
        ssum = ssum * ex2f(m - mr) + so * ex2f(mo - mr);
        m = mm;
      };
      if (tq >= 2) { pm[(tq - 2) * 128 + lc] = m; ps[(tq - 2) * 128 + lc] = ssum; }
      named_bar(1, kCP1Warps * 32);
      if (tq < 2) merge(pm[tq * 128 + lc], ps[tq * 128 + lc]);
      named_bar(1, kCP1Warps * 32);
      if (tq == 1) { pm[lc] = m; ps[lc] = ssum; }
      named_bar(1, kCP1Warps * 32);
      if (tq == 0 && col_ok) {
        merge(pm[lc], ps[lc]);
        a.part[((size_t)A.unit * a.cmax + A.ci) * K::GW + gcol] = ssum > 0.f ? m + lg2f(ssum) : -INFINITY;
      }
      named_bar(1, kCP1Warps * 32);
      if (warp == kCEpi0 && lane == 0) {
        if (jp < 2048) CTRACE(40960 + 2 * jp, clk32());
        mbar_arrive(p1pub0 + 8 * (jp & 3));   // the combiner publishes them (counter release)
      }
    }
  } else {
    // ================= pass-2 warps (4): token t = tile*256 + rank*128 + q*32 + lane, all window rows of
    // the pass-2 accumulator (B_aug already subtracted L2/s), in chunks of RC rows
    const int q = warp & 3;
    const uint32_t tbase2 = tmem + ((uint32_t)(q * 32) << 16) + 256;
    // half h (buffer 256 + h*GWH) holds, per token, window rows h*W/4 .. +W/4 (rank 0's Q rows) then
    // W/2 + h*W/4 .. +W/4 (rank 1's)
    constexpr int RQ = W / 4;
    constexpr int RC = G >= 7 ? 4 : 8;   // rows per TMEM load chunk
    static_assert(RQ % RC == 0, "chunking");
    int n2 = 0;
    for (int jq = 0;; ++jq) {
      mbar_wait(ctabf0 + 8 * (jq & 7), (uint32_t)((jq >> 3) & 1));
      Chunk B;
      {
        const volatile int* ce = ctab + kCtabInts * (jq & 7);
        B.unit = ce[5];
        if (B.unit < 0) break;
        B.T = ce[0]; B.tb = ce[4]; B.nt = ce[8];
      }
      for (int k = 0; k < B.nt; ++k, ++n2) {
        const int t = (B.tb + p2_tile(k, B.nt)) * 2 * kTile + rank * kTile + q * 32 + lane;
        const int du = t - (B.T - W);   // window row u contributes iff u >= du (token t <= T-w+u)
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          mbar_wait_lean(accf0 + 8 * (2 + h), (uint32_t)(n2 & 1));
          tc_fence_after();
          if (CDEBUG(2)) {   // bisection: no pass-2 math
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_remote_arrive_relaxed(acce0 + 8 * (2 + h), 0);
            continue;
          }
#pragma unroll
          for (int ch = 0; ch < 2 * RQ / RC; ++ch) {
            float v[RC * G];
#pragma unroll
            for (int kk = 0; kk < RC * G / 4; ++kk) TMEM_LD4(tbase2 + h * K::GWH + ch * RC * G + kk * 4, v, kk * 4);
            tmem_wait_ld();
            if (ch + 1 == 2 * RQ / RC) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_remote_arrive_relaxed(acce0 + 8 * (2 + h), 0);
            }
            const int ubase = (ch * RC / RQ) * (W / 2) + h * RQ + (ch * RC) % RQ;
#pragma unroll
            for (int r = 0; r < RC; ++r) {
              const float* y = v + r * G;
              float mx;
              if constexpr (G == 7) mx = max3f(max3f(y[0], y[1], y[2]), max3f(y[3], y[4], y[5]), y[6]);
              else if constexpr (G == 8) mx = max3f(max3f(y[0], y[1], y[2]), max3f(y[3], y[4], y[5]), fmaxf(y[6], y[7]));
              else if constexpr (G == 5) mx = max3f(max3f(y[0], y[1], y[2]), y[3], y[4]);
              else {
                mx = y[0];
#pragma unroll
                for (int g = 1; g < G; ++g) mx = fmaxf(mx, y[g]);
              }
              const float pterm = ex2f(mx * scale);
              acc[r & 3] += (ubase + r >= du) ? pterm : 0.f;
            }
          }
        }
        if (t < B.T)
          c.ws.scores[(size_t)B.unit * c.max_seq_len + t] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) * (1.0f / W);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();   // the peer's MMAs / remote arrivals are over before TMEM is released
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ------------------------------------------------------------------ host side
#ifdef ZPC_TUNING
uint32_t* g_trace = nullptr;   // tuning builds only (the production library keeps no global state)
#endif
template <int G, int W, int D>
cudaError_t launch_coop_t(const Call& c, cudaStream_t s) {
  using K = CfgC<G, W, D>;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  // Q cache viewed as [rows = L*M*w][h_q][d]; one box = the unit's G heads x w/2 window rows (a CTA's half)
  CUtensorMap tq;
  const cuuint32_t estr[3] = {1, 1, 1};
  const cuuint64_t qdim[3] = {(cuuint64_t)c.d, (cuuint64_t)c.h_q, (cuuint64_t)c.L * c.M * c.w};
  const cuuint64_t qstr[2] = {(cuuint64_t)c.d * 2, (cuuint64_t)c.h_q * c.d * 2};
  const cuuint32_t qbox[3] = {64, (cuuint32_t)G, (cuuint32_t)(W / 2)};
  if (enc(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(c.q_cache), qdim, qstr, qbox, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  // K as [rows = L*N_total*b][h_kv][d]; one box = min(b, 128) consecutive slots x 64 elements of one head
  CUtensorMap tk;
  memset(&tk, 0, sizeof(tk));
  int ktma = 0;
#ifndef ZPC_COOP_TMA
#define ZPC_COOP_TMA 1
#endif
  // only for blocks of >= 128 slots: with b = 16 a tile is 16 boxes of 16 rows per CTA and the TMA path measured
  // 15.0 ms on the qwen7b batch against 8.2-8.5 for the cp.async gather (tuning build, one B200)
  if (ZPC_COOP_TMA && c.b >= 128 && c.b <= 256 && (c.b & (c.b - 1)) == 0) {
    const cuuint64_t kdim[3] = {(cuuint64_t)c.d, (cuuint64_t)c.h_kv, (cuuint64_t)c.L * c.N_total * c.b};
    const cuuint64_t kstr[2] = {(cuuint64_t)c.d * 2, (cuuint64_t)c.h_kv * c.d * 2};
    const cuuint32_t kbox[3] = {64, 1, (cuuint32_t)std::min(c.b, kTile)};
    ktma = enc(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, c.k_cache, kdim, kstr, kbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
  }
  auto kern = k_score_coop<G, W, D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // every pair must be co-resident (pairs wait on each other's chunks): one CTA per SM, as many pairs as
  // the occupancy query allows at once
  int dev = 0, sms = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  int npairs = sms / 2;
  cfg.gridDim = dim3(2);
  int q = 0;
  if (cudaOccupancyMaxActiveClusters(&q, kern, &cfg) == cudaSuccess && q > 0) npairs = std::min(npairs, q);
  cudaGetLastError();
  CoopArgs ca;
  const int npt_max = (c.max_seq_len + 255) / 256;
  int kt = ZPC_COOP_KT;
  ca.delta = ZPC_COOP_DELTA;
  ca.hints = ZPC_COOP_HINTS;
  ca.debug = 0;
#ifdef ZPC_TUNING   // A/B builds only: the production library reads no environment
  if (const char* e = getenv("ZPC_COOP_KT")) kt = std::max(kCoopChunkTiles, atoi(e));
  if (const char* e = getenv("ZPC_COOP_DELTA")) ca.delta = atoi(e);
  if (const char* e = getenv("ZPC_COOP_HINTS")) ca.hints = atoi(e);
  if (const char* e = getenv("ZPC_COOP_DEBUG")) ca.debug = atoi(e);
#endif
  ca.kt = std::max(kt, (npt_max + npairs - 1) / npairs);   // chunks per unit <= pairs
  ca.trace = nullptr;
#ifdef ZPC_TUNING
  if (getenv("ZPC_COOP_TRACE")) {
    if (!g_trace) cudaMalloc(&g_trace, 49152 * 4);
    cudaMemsetAsync(g_trace, 0, 49152 * 4, s);
    ca.trace = g_trace;
  }
#endif
  // (l, h)-major order for shared-prefix calls measured SLOWER on the prefix config (score 25.7 -> 30.5 ms,
  // L2 hit 21%): ~24 pairs reading the same prefix lines at the same moment concentrate on a few L2 slices.
  // Kept as a tuning switch; the dedup that pays needs the prefix tiles multiplied once against all the
  // sharing requests' queries.
  ca.lh_major = 0;
  ca.ktma = ktma;
#ifdef ZPC_TUNING
  if (const char* e = getenv("ZPC_COOP_KTMA")) ca.ktma = std::min(ktma, atoi(e));
#endif
#ifdef ZPC_TUNING
  if (const char* e = getenv("ZPC_COOP_LHMAJOR")) ca.lh_major = atoi(e);
#endif
  ca.cmax = c.ws.coop_cmax;
  ca.npairs = npairs;
  ca.part = c.ws.coop_part;
  ca.cnt = c.ws.coop_cnt;
  ca.rs = c.ws.coop_rs;
  k_coop_plan<<<1, 1024, 0, s>>>(c, ca);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cfg.gridDim = dim3((unsigned)(2 * npairs));
  return cudaLaunchKernelEx(&cfg, kern, c, ca, tq, tk);
}

template <int D>
cudaError_t dispatch_coop(const Call& c, cudaStream_t s, bool* used) {
  *used = true;
  switch (c.G) {
    case 5: return launch_coop_t<5, 32, D>(c, s);
    case 7: return launch_coop_t<7, 32, D>(c, s);
    case 8: return launch_coop_t<8, 32, D>(c, s);
    default: *used = false; return cudaSuccess;
  }
}

}  // namespace

// Two-pass bf16 calls with w = 32 and G*w/2 in (64, 128] (G = 5, 7, 8): the cooperative pair kernel.
// Others (single-pass ZPC_F_LSE_INPUT, w = 16, G = 4) fall through to launch_score_tc.
bool score_coop_applies(const Call& c) {
  if (c.dtype != ZPC_BF16 || c.lse_in != nullptr || c.w != 32 || (c.variant & ZPC_V_SCORE_SERIAL)) return false;
  if (c.d != 64 && c.d != 128) return false;
  if (c.b < 5) return false;   // a 128-token tile must span <= kMaxIds blocks
  return c.G == 5 || c.G == 7 || c.G == 8;
}

cudaError_t launch_score_coop(const Call& c, cudaStream_t s, bool* used) {
  *used = false;
  if (!score_coop_applies(c)) return cudaSuccess;
  if (c.R * c.L * c.h_kv == 0) { *used = true; return cudaSuccess; }
  return c.d == 64 ? dispatch_coop<64>(c, s, used) : dispatch_coop<128>(c, s, used);
}

}  // namespace zpc

#ifdef ZPC_TUNING
extern "C" int zpc_debug_trace_copy(void* host, size_t bytes) {
  if (!zpc::g_trace) return -1;
  return cudaMemcpy(host, zpc::g_trace, bytes < 49152 * 4 ? bytes : 49152 * 4, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}
#endif
