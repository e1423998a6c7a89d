// tcgen05.mma (kind::f16, bf16 -> fp32, both operands SW128 K-major in shared memory) throughput
// for the score kernel's shapes: cycles per instruction, one CTA per SM, one issuing thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ub scripts/umma_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int N, int KSTEPS, int REPS, int RD>
__global__ void __launch_bounds__(128 + 256, 1) k(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) stop = 0;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3F803F80u, 0, 0, 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp >= 4) {
    // RD reader warps (warps 4..4+RD-1): stream tcgen05.ld 32x32b.x16 over columns 256..511 (the other accumulator)
    if (warp - 4 < RD) {
      const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + 256;
      float acc = 0.f;
      uint32_t v[16];
      for (int it = 0; !stop; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                         "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                       : "r"(base + ((it * 8 + c) & 15) * 16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) acc += __uint_as_float(v[j]);
        }
      }
      if (acc == 1234.5f) out[1] = 1;
    }
  } else if (threadIdx.x == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(smem);             // A: 128 rows, 2 slabs of 16 KB
    const uint32_t b0 = a0 + 32 * 1024;                                       // B: N rows, 2 slabs of N*128 B
    const uint32_t bb = (uint32_t)__cvta_generic_to_shared(&bar);
    long long t0 = clock64();
    for (int r = 0; r < REPS; ++r) {
      const uint32_t d = slot;
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk)
        umma(d, sw128_desc(a0 + (kk >> 2) * 16384 + (kk & 3) * 32), sw128_desc(b0 + (kk >> 2) * N * 128 + (kk & 3) * 32),
             idesc_bf16(128, N), kk > 0);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bb) : "memory");
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(bb) : "memory");
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}


// issue-queue probe: time to issue n MMAs (N=224) into an idle pipe, and to completion
__global__ void __launch_bounds__(128, 1) kq(unsigned long long* out, int n) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3F803F80u, 0, 0, 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(smem), b0 = a0 + 32 * 1024;
    const uint32_t bb = (uint32_t)__cvta_generic_to_shared(&bar);
    long long t0 = clock64();
    for (int r = 0; r < n; ++r)
      umma(slot, sw128_desc(a0 + (r & 3) * 32), sw128_desc(b0 + (r & 3) * 32), idesc_bf16(128, 224), r > 0);
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bb) : "memory");
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(bb) : "memory");
    }
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int N, int KSTEPS, int RD>
void run() {
  constexpr int REPS = 2000;
  unsigned long long* o; cudaMalloc(&o, 16);
  cudaFuncSetAttribute(k<N, KSTEPS, REPS, RD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(a); k<N, KSTEPS, REPS, RD><<<148, 128 + 256, 200 * 1024>>>(o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  unsigned long long cyc; cudaMemcpy(&cyc, o, 8, cudaMemcpyDeviceToHost);
  const double per = (double)cyc / (REPS * KSTEPS);
  const double flop = 2.0 * 128 * N * 16;
  printf("readers %d M=128 N=%3d K=16: %6.1f cycles/MMA (ideal 8192 flop/clk: %5.1f) -> %5.0f flop/clk/SM; all SMs %.0f TFLOP/s (%s)\n", RD, N, per,
         flop / 8192, flop / per, 148.0 * flop * REPS * KSTEPS / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned long long* o; cudaMalloc(&o, 16);
  cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int n : {1, 2, 3, 4, 6, 8, 9, 12, 16, 32}) {
    unsigned long long h[2];
    for (int r = 0; r < 2; ++r) { kq<<<148, 128, 200 * 1024>>>(o, n); cudaDeviceSynchronize(); }
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("issue %2d MMAs (128x224x16): issue %6llu cycles, complete %6llu cycles\n", n, h[0], h[1]);
  }
  return 0;
}
