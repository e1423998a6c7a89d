// How often does a waiting warp poll? One warp waits ~100 us on an mbarrier that another warp
// completes; count the waiter's loop iterations for several wait idioms.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wb scripts/wait_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t try_wait(uint32_t bar, uint32_t par) {
  uint32_t d;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(d) : "r"(bar), "r"(par) : "memory");
  return d;
}
__device__ __forceinline__ uint32_t try_wait_hint(uint32_t bar, uint32_t par, uint32_t ns) {
  uint32_t d;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(d) : "r"(bar), "r"(par), "r"(ns) : "memory");
  return d;
}
__device__ __forceinline__ uint32_t test_wait(uint32_t bar, uint32_t par) {
  uint32_t d;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(d) : "r"(bar), "r"(par) : "memory");
  return d;
}

template <int M>
__global__ void k(unsigned long long* out, long long work_cycles) {
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  __syncthreads();
  const int warp = threadIdx.x / 32;
  if (warp == 1) {
    const long long t0 = clock64();
    while (clock64() - t0 < work_cycles) {}
    if (threadIdx.x == 32) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
  } else if (warp == 0) {
    unsigned long long it = 0;
    const long long t0 = clock64();
    while (true) {
      ++it;
      uint32_t d;
      if (M == 0) d = try_wait(b, 0);
      else if (M == 1) d = try_wait_hint(b, 0, 1000000);
      else if (M == 2) { d = try_wait(b, 0); if (!d) __nanosleep(2000); }
      else if (M == 3) { d = test_wait(b, 0); if (!d) __nanosleep(2000); }
      else if (M == 4) { d = test_wait(b, 0); if (!d) __nanosleep(100000); }
      else { d = try_wait_hint(b, 0, 0x7fffffff); }
      if (d) break;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = it; out[1] = t1 - t0; }
  }
}
template <int M>
void run(const char* name) {
  unsigned long long* o; cudaMalloc(&o, 16);
  unsigned long long h[2];
  k<M><<<1, 64>>>(o, 200000);   // ~100 us at ~1.9 GHz
  cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("%-34s iterations %8llu over %8llu cycles -> %.1f cycles/iter (%s)\n", name, h[0], h[1], (double)h[1] / h[0],
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("try_wait (no hint)");
  run<1>("try_wait hint 1e6 ns");
  run<5>("try_wait hint 0x7fffffff");
  run<2>("try_wait + nanosleep(2000)");
  run<3>("test_wait + nanosleep(2000)");
  run<4>("test_wait + nanosleep(100000)");
  return 0;
}
