#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#ifndef POLY
#define POLY 0
#endif
#ifndef POLYDEN
#define POLYDEN 4
#endif
constexpr bool kPolyOffload = POLY != 0;
__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
#define TMEM_LD16(taddr, v, off) asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
  : "=f"(v[off+0]),"=f"(v[off+1]),"=f"(v[off+2]),"=f"(v[off+3]),"=f"(v[off+4]),"=f"(v[off+5]),"=f"(v[off+6]),"=f"(v[off+7]),"=f"(v[off+8]),"=f"(v[off+9]),"=f"(v[off+10]),"=f"(v[off+11]),"=f"(v[off+12]),"=f"(v[off+13]),"=f"(v[off+14]),"=f"(v[off+15]) : "r"(taddr))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
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
template <int N>
__device__ __forceinline__ float sum_exp_n(const float* v, float scale, float m) {
  uint64_t acc[4] = {0, 0, 0, 0};
  const uint64_t S2 = pk2(scale, scale), NM2 = pk2(-m, -m);
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const uint64_t arg = fma2(pk2(v[2 * j], v[2 * j + 1]), S2, NM2);
    if (kPolyOffload && (j % POLYDEN) < POLY) {
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

template <int WARPS, int NB, int LOADERS>
__global__ void __launch_bounds__((WARPS + LOADERS) * 32, 1) k(float* out, int steps, const int4* gsrc, size_t gsz) {
  __shared__ uint32_t slot;
  extern __shared__ __align__(1024) uint8_t ring[];
  if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t*>(ring + 99 * 1024) = 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp >= WARPS && LOADERS == 8) {   // idle warps: just wait for the end
    volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>(ring + 99 * 1024);
    while (*flag == 0) __nanosleep(1000);
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
    return;
  }
  if (warp >= WARPS) {   // loaders: stream 16-B cp.async (1 KB-strided rows) into a 96 KB smem ring until told to stop
    const int lt = threadIdx.x - WARPS * 32;
    size_t pos = ((size_t)blockIdx.x * 7919 + lt) * 64;
    volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>(ring + 99 * 1024);
    for (int it = 0; it < (1 << 30) && *flag == 0; ++it) {
      for (int k = 0; k < 16; ++k) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring) + (uint32_t)(((it * 16 + k) * LOADERS * 32 + lt) % 6144) * 16;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gsrc + (pos % gsz)) : "memory");
        pos += 64 * 16 + 1;
      }
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group 2;");
    }
    asm volatile("cp.async.wait_all;");
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
    return;
  }
  const int q = warp & 3, half = (warp >> 2) & 1;
  const uint32_t lane_base = slot + ((uint32_t)(q * 32) << 16) + half * 128 + ((warp >> 3) & 1) * 0;
  const float scale = 0.1275f;
  float m = 3.0f, ssum = 0.f;
  for (int st = 0; st < steps; ++st) {
    const int a = st & 1;
    float vb[2][NB];
    TMEM_LD16(lane_base + a * 256, vb[0], 0);
    if (NB == 32) TMEM_LD16(lane_base + a * 256 + 16, vb[0], 16);
#pragma unroll
    for (int bh = 0; bh < 128 / NB; ++bh) {
      float* v = vb[bh & 1];
      tmem_wait_ld();
      if (bh + 1 < 128 / NB) {
        TMEM_LD16(lane_base + a * 256 + (bh + 1) * NB, vb[(bh + 1) & 1], 0);
        if (NB == 32) TMEM_LD16(lane_base + a * 256 + (bh + 1) * NB + 16, vb[(bh + 1) & 1], 16);
      }
      float bsum = sum_exp_n<NB>(v, scale, m);
      if (!(bsum < 1.8446744e19f)) { m += 1.f; }
      ssum += bsum;
    }
  }
  if (ssum == 1234.5f) out[0] = ssum;
  if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t*>(ring + 99 * 1024) = 1;
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
template <int WARPS, int NB, int LOADERS>
void run() {
  float* out; cudaMalloc(&out, 4);
  static int4* gsrc = nullptr; const size_t gsz = (size_t)1 << 28;
  if (!gsrc) { cudaMalloc(&gsrc, gsz * 16); cudaMemset(gsrc, 0, gsz * 16); }
  cudaFuncSetAttribute(k<WARPS, NB, LOADERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int steps = 3000; float ms = 0;
  for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k<WARPS, NB, LOADERS><<<148, (WARPS + LOADERS) * 32, 100 * 1024>>>(out, steps, gsrc, gsz); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); }
  printf("pass-1 step replica: %2d warps NB=%d loaders=%d: %.3f us/step (%s)\n", WARPS, NB, LOADERS, ms * 1e3 / steps, cudaGetErrorString(cudaGetLastError()));
}
int main() { run<8, 32, 0>(); run<8, 32, 8>(); return 0; }
