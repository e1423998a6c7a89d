// tcgen05.ld throughput: W warps per CTA (1 CTA/SM) repeatedly load 32x32b.xN and wait.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define LD16(taddr, v, off) asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
  : "=f"(v[off+0]),"=f"(v[off+1]),"=f"(v[off+2]),"=f"(v[off+3]),"=f"(v[off+4]),"=f"(v[off+5]),"=f"(v[off+6]),"=f"(v[off+7]),"=f"(v[off+8]),"=f"(v[off+9]),"=f"(v[off+10]),"=f"(v[off+11]),"=f"(v[off+12]),"=f"(v[off+13]),"=f"(v[off+14]),"=f"(v[off+15]) : "r"(taddr))
template <int NLD>
__global__ void __launch_bounds__(256, 1) k(float* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    float v[NLD * 16];
#pragma unroll
    for (int j = 0; j < NLD; ++j) LD16(base + j * 16, v, j * 16);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < NLD * 16; ++j) acc += v[j];
  }
  if (acc == 1234.5f) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
template <int NLD>
void run() {
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000; float ms = 0;
  for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k<NLD><<<148, 256>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); }
  const double bytes_per_sm = 256.0 * NLD * 16 * 4 * iters;
  printf("tcgen05.ld x16 * %d per wait, 8 warps: %.3f ms -> %.1f B/clk/SM (%s)\n", NLD, ms, bytes_per_sm / (ms * 1e-3) / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}
int main() { run<1>(); run<4>(); run<8>(); return 0; }
