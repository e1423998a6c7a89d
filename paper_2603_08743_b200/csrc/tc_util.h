// PTX wrappers shared by the tcgen05 scoring kernels (score_tc.cu, score_coop.cu): mbarriers, TMA,
// cp.async, tcgen05 MMA / commit / TMEM loads, cluster barriers, packed fp32x2 math, the tensor-map
// encoder entry point. Library-private; each including TU gets its own internal-linkage copy.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include "internal.h"

namespace zpc {
namespace {

constexpr int kTile = 128;       // tokens per tile (UMMA M in pass 2, N in pass 1)
constexpr int kIdSlots = 8;      // block-id ring of the feeder warp (tiles in flight + 2 being read)
constexpr int kIdAhead = 4;      // tiles whose ids the feeder has in flight ahead of the published one
constexpr int kMaxIds = 32;      // block ids per 128-token tile (b >= 5)
constexpr uint32_t kTmemCols = 512;
constexpr float kLog2e = 1.4426950408889634f;
#ifndef ZPC_WAIT_HINT_NS
#define ZPC_WAIT_HINT_NS 1000000   // mbarrier try_wait suspend-time hint (0 = none)
#endif

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// %globaltimer in ns: waits trap after kWaitLimitNs so a pipeline bug fails loudly instead of hanging
constexpr unsigned long long kWaitLimitNs = 10ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// a pipeline wait that exceeded kWaitLimitNs: report which barrier (tuning builds) and trap
__device__ __noinline__ void wait_trap(uint32_t bar, uint32_t parity) {
#ifdef ZPC_DEBUG_WAITS
  printf("zpc wait timeout: block %d warp %d bar smem+%u parity %u\n", blockIdx.x, threadIdx.x / 32, bar, parity);
#endif
  __trap();
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
  unsigned long long t_start = 0;
  while (true) {
#if ZPC_WAIT_HINT_NS > 0
    // suspend-time hint: the thread sleeps until the phase completes (or the hint), no busy polling
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(ZPC_WAIT_HINT_NS)
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
#endif
    if (done) return;
    if (spins++ == 0) t_start = gtime_ns();
    else if ((spins & 15) == 0 && gtime_ns() - t_start > kWaitLimitNs) wait_trap(bar, parity);   // fail loudly, never hang
  }
}
// epilogue waiters that share an SMSP with working warps (k_score_coop's pass-1 / pass-2 warps): try_wait
// without a suspend-time hint in a lean loop -- a 32-bit poll counter is the hang detector (2^22 polls, ~16 s)
// instead of a 64-bit counter and a %globaltimer branch per poll. Measured (A/B on one B200): k_score_coop
// qwen7b 7.53 -> 7.42 ms, k_score_tc --lse-input 3.60 -> 3.53, k_score_ovl llama8b 11.96 -> 11.92; k_score_res
// paper_op 0.1758 -> 0.1765 (kept on mbar_wait); the same loop for every wait of every kernel 7.75 -> 9.07 ms
// (producers without the hint spin); the MMA issuers' and feeders' waits alone through lean loops: qwen7b
// 7.57 -> 8.60, llama8b 12.1 -> 12.9 (their waits keep the hint).
__device__ __forceinline__ void mbar_wait_lean(uint32_t bar, uint32_t parity) {
  for (uint32_t n = 0;; ++n) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (n == (1u << 22)) wait_trap(bar, parity);   // a failed try_wait suspends ~4 us (scripts/trywait_probe.cu): ~16 s
  }
}
// for waiters off the critical path: back off between polls so they do not flood the issue
// slots / instruction cache the MUFU-bound epilogue needs (measured: polls were 19% no_inst)
__device__ __forceinline__ void mbar_wait_backoff(uint32_t bar, uint32_t parity, int ns) {
  uint32_t done = 0;
  long long spins = 0;
  unsigned long long t_start = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(ns);
    if (spins++ == 0) t_start = gtime_ns();
    else if ((spins & 15) == 0 && gtime_ns() - t_start > kWaitLimitNs) wait_trap(bar, parity);
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
__device__ __forceinline__ int lds_s32(uint32_t addr) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// the mbarrier counts this thread's arrival once all its prior cp.async have landed
// debug timeline stamp (ZPC_SCORE_DEBUG bit 1; CTA 0 only): SM cycle counter (%globaltimer ticks too coarsely)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
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
// no-swizzle K-major descriptor (core matrices 8 rows x 16 B): LBO = K-direction core-matrix
// stride, SBO = M/N-direction 8-row-group stride
__device__ __forceinline__ uint64_t none_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                      // descriptor version (sm_100); layout 0 = no swizzle
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
// issued by one elected lane of a converged warp (operands warp-uniform -> uniform registers)
__device__ __forceinline__ void umma_elect(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
      : "memory");
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
__device__ __forceinline__ void named_bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
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

// ------------------------------------------------------------------ packed fp32x2 + misc helpers
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// packed 2^x, x <= 0, on the FMA pipe (see ex2_poly)
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x2) {
  float x0, x1;
  upk2(x2, x0, x1);
  x2 = pk2(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
  const uint64_t t2 = add2(x2, pk2(12582912.f, 12582912.f));
  const uint64_t n2 = add2(t2, pk2(-12582912.f, -12582912.f));
  const uint64_t f2 = fma2(n2, pk2(-1.f, -1.f), x2);
  uint64_t p = fma2(pk2(1.3534167e-4f, 1.3534167e-4f), f2, pk2(1.3395720e-3f, 1.3395720e-3f));
  p = fma2(p, f2, pk2(9.6180239e-3f, 9.6180239e-3f));
  p = fma2(p, f2, pk2(5.5504109e-2f, 5.5504109e-2f));
  p = fma2(p, f2, pk2(2.4022652e-1f, 2.4022652e-1f));
  p = fma2(p, f2, pk2(6.9314718e-1f, 6.9314718e-1f));
  p = fma2(p, f2, pk2(1.0f, 1.0f));
  float p0, p1, t0, t1;
  upk2(p, p0, p1);
  upk2(t2, t0, t1);
  // (bits(t) - bits(1.5*2^23)) << 23 == bits(t) << 23 (mod 2^32): the magic's low 9 bits are 0
  return pk2(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
             __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}
// packed 2^x on the FMA pipe, degree-4 minimax on the Cody-Waite remainder f in [-0.5, 0.5]
// (max relative error 2.7e-6 in fp32, measured on a 2e5-point grid): 7 FFMA2/FADD2 + 4 ALU per pair.
// Callers pass x <= 0 (arguments relative to a running maximum); x is clamped below at -126 so the
// exponent never wraps (masked -inf arguments give 2^-126, below fp32 resolution of any sum >= 1).
__device__ __forceinline__ uint64_t ex2_poly4x2(uint64_t x2) {
  float x0, x1;
  upk2(x2, x0, x1);
  x2 = pk2(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t t2 = add2(x2, pk2(12582912.f, 12582912.f));     // 1.5 * 2^23: round to nearest integer
  const uint64_t n2 = add2(t2, pk2(-12582912.f, -12582912.f));
  const uint64_t f2 = fma2(n2, pk2(-1.f, -1.f), x2);
  uint64_t p = fma2(pk2(0.009570134803652763f, 0.009570134803652763f), f2, pk2(0.05591796338558197f, 0.05591796338558197f));
  p = fma2(p, f2, pk2(0.240247443318367f, 0.240247443318367f));
  p = fma2(p, f2, pk2(0.6931217908859253f, 0.6931217908859253f));
  p = fma2(p, f2, pk2(0.9999992847442627f, 0.9999992847442627f));
  float p0, p1, t0, t1;
  upk2(p, p0, p1);
  upk2(t2, t0, t1);
  // (bits(t) - bits(1.5*2^23)) << 23 == bits(t) << 23 (mod 2^32): the magic's low 9 bits are 0
  return pk2(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
             __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}
__device__ __forceinline__ void mbar_remote_arrive(uint32_t local_bar, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_bar), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
// relaxed remote arrival: for accumulator releases, ordered by tcgen05.wait::ld + fence::before_thread_sync
// (a release here would also wait for the warp's outstanding global stores to become cluster-visible)
__device__ __forceinline__ void mbar_remote_arrive_relaxed(uint32_t local_bar, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_bar), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  long long spins = 0;
  unsigned long long t_start = 0;
  while (true) {
#if ZPC_WAIT_HINT_NS > 0
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(ZPC_WAIT_HINT_NS)
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
#endif
    if (done) return;
    if (spins++ == 0) t_start = gtime_ns();
    else if ((spins & 15) == 0 && gtime_ns() - t_start > kWaitLimitNs) wait_trap(bar, parity);
  }
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

#define TMEM_LD8(taddr, v, off)                                                                           \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                 \
               : "=f"(v[off + 0]), "=f"(v[off + 1]), "=f"(v[off + 2]), "=f"(v[off + 3]), "=f"(v[off + 4]),  \
                 "=f"(v[off + 5]), "=f"(v[off + 6]), "=f"(v[off + 7])                                     \
               : "r"(taddr))
#define TMEM_LD4(taddr, v, off)                                                                           \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"                               \
               : "=f"(v[off + 0]), "=f"(v[off + 1]), "=f"(v[off + 2]), "=f"(v[off + 3])                   \
               : "r"(taddr))

__device__ __forceinline__ void umma2_elect(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// commit to the barrier at this smem offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma2_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n"
      ::"r"(bar), "h"((uint16_t)3)
      : "memory");
}

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

}  // namespace
}  // namespace zpc
