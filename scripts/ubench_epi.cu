// Round-2 microbenchmarks for the score-kernel epilogue budget on one B200 (one CTA per SM, 148 CTAs):
//  (1) tcgen05.ld throughput (32x32b.xN) vs warps per CTA, (2) MUFU ex2, FFMA2/FADD2 with register
//  operands, (3) a pass-1-like loop (LDTM -> FMUL2 -> ex2 -> FADD2) in elements/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LDX32(taddr, v, off)                                                                                 \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                      \
               : "=f"(v[off + 0]), "=f"(v[off + 1]), "=f"(v[off + 2]), "=f"(v[off + 3]), "=f"(v[off + 4]),     \
                 "=f"(v[off + 5]), "=f"(v[off + 6]), "=f"(v[off + 7]), "=f"(v[off + 8]), "=f"(v[off + 9]),     \
                 "=f"(v[off + 10]), "=f"(v[off + 11]), "=f"(v[off + 12]), "=f"(v[off + 13]), "=f"(v[off + 14]), \
                 "=f"(v[off + 15]), "=f"(v[off + 16]), "=f"(v[off + 17]), "=f"(v[off + 18]), "=f"(v[off + 19]), \
                 "=f"(v[off + 20]), "=f"(v[off + 21]), "=f"(v[off + 22]), "=f"(v[off + 23]), "=f"(v[off + 24]), \
                 "=f"(v[off + 25]), "=f"(v[off + 26]), "=f"(v[off + 27]), "=f"(v[off + 28]), "=f"(v[off + 29]), \
                 "=f"(v[off + 30]), "=f"(v[off + 31])                                                         \
               : "r"(taddr))
#define LDX16(taddr, v, off)                                                                                 \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=f"(v[off + 0]), "=f"(v[off + 1]), "=f"(v[off + 2]), "=f"(v[off + 3]), "=f"(v[off + 4]),     \
                 "=f"(v[off + 5]), "=f"(v[off + 6]), "=f"(v[off + 7]), "=f"(v[off + 8]), "=f"(v[off + 9]),     \
                 "=f"(v[off + 10]), "=f"(v[off + 11]), "=f"(v[off + 12]), "=f"(v[off + 13]), "=f"(v[off + 14]), \
                 "=f"(v[off + 15])                                                                             \
               : "r"(taddr))

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint64_t pk2(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) { uint64_t d; asm volatile("mul.rn.f32x2 %0,%1,%2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t d; asm volatile("add.rn.f32x2 %0,%1,%2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm volatile("fma.rn.f32x2 %0,%1,%2,%3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

__device__ uint32_t g_slot[148];

// MODE 0: LDTM x32 only; 1: LDTM x16 only; 2: pass-1 loop (LDTM x32 -> mul2 -> ex2 -> add2)
// 3: pass-1 loop without the LDTM (values from registers); 4: MUFU ex2 only; 5: FFMA2 reg operands only
// 6: FADD2 only
template <int MODE, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k(float* out, int iters, float sc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (MODE <= 2) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  const uint32_t base = (MODE <= 2 ? slot : 0u) + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32) % 512;
  uint64_t acc[4] = {0, 0, 0, 0};
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = -0.001f * (threadIdx.x + j);
  const uint64_t s2 = pk2(sc, sc);
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0 || MODE == 2) { LDX32(base + (i & 7) * 32, v, 0); asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
    if (MODE == 1) { LDX16(base + (i & 15) * 16, v, 0); LDX16(base + ((i + 1) & 15) * 16, v, 16); asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
    if (MODE == 0 || MODE == 1) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) acc[j / 8] = add2(acc[j / 8], pk2(v[j], v[j + 1]));
    }
    if (MODE == 2 || MODE == 3) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        uint64_t a = mul2(pk2(v[2 * j], v[2 * j + 1]), s2);
        float a0, a1; upk2(a, a0, a1);
        acc[j & 3] = add2(acc[j & 3], pk2(ex2(a0), ex2(a1)));
      }
      if (MODE == 3) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += 1e-7f;
      }
    }
    if (MODE == 4) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = ex2(v[j]);
    }
    if (MODE == 5) {
#pragma unroll
      for (int j = 0; j < 16; ++j) { uint64_t a = fma2(pk2(v[2 * j], v[2 * j + 1]), s2, acc[j & 3]); upk2(a, v[2 * j], v[2 * j + 1]); }
    }
    if (MODE == 6) {
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j & 3] = add2(acc[j & 3], pk2(v[2 * j], v[2 * j + 1]));
    }
  }
  float a0 = 0, a1 = 0, s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) { upk2(acc[j], a0, a1); s += a0 + a1; }
#pragma unroll
  for (int j = 0; j < 32; ++j) s += v[j];
  if (s == 1234.5f) out[0] = s;
  if (MODE <= 2) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  }
}

template <int MODE, int NW>
void run(const char* name) {
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  float ms = 0;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    k<MODE, NW><<<148, NW * 32>>>(out, iters, 0.999f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  const double elems_per_sm = (double)NW * 32 * 32 * iters;   // 32 fp32 values per thread per iter
  const double clk = ms * 1e-3 * 1.965e9;                      // assumes the max SM clock
  printf("%-34s warps=%2d %8.3f ms  %7.2f elem/clk/SM  %7.1f B/clk/SM  (%s)\n", name, NW, ms, elems_per_sm / clk,
         elems_per_sm * 4 / clk, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0, 4>("LDTM 32x32b.x32");
  run<0, 8>("LDTM 32x32b.x32");
  run<0, 16>("LDTM 32x32b.x32");
  run<1, 8>("LDTM 32x32b.x16 x2");
  run<1, 16>("LDTM 32x32b.x16 x2");
  run<2, 8>("pass1 loop LDTM+mul2+ex2+add2");
  run<2, 16>("pass1 loop LDTM+mul2+ex2+add2");
  run<3, 8>("pass1 loop regs mul2+ex2+add2");
  run<3, 16>("pass1 loop regs mul2+ex2+add2");
  run<4, 8>("MUFU ex2 only");
  run<4, 16>("MUFU ex2 only");
  run<5, 16>("FFMA2 reg operands");
  run<6, 16>("FADD2");
  return 0;
}
