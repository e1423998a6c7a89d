// Bisection microbenchmark: the score kernel's K-ring structure without MMA/epilogue math.
// Variants (template MODE bits): 1 = relay through a separate thread (MMA-like) before refill,
// 2 = two passes per unit (pass 2 reversed), 4 = runtime block size (division), 8 = big smem (210 KB)
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int L = 28, HKV = 4, D = 128, R = 64, T = 8192;
constexpr int NB = T / 16, NT = R * NB + 64, TILE = 128, STAGE = TILE * D * 2, ST = 3;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint32_t b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n)); }
__device__ __forceinline__ void marrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void mwait(uint32_t b, uint32_t ph) {
  uint32_t d = 0;
  while (!d) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(d) : "r"(b), "r"(ph) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(352, 1) ring(const uint16_t* K, const int* tables, int units, int bsz, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + ST * STAGE + 64);
  const uint32_t full0 = su(bars), relay0 = su(bars + ST);
  if (threadIdx.x == 0) { for (int s = 0; s < ST; ++s) { minit(full0 + 8 * s, 256); minit(relay0 + 8 * s, 1); } minit(relay0 + 8 * ST, 1); }
  __syncthreads();
  const int ntile = T / TILE;
  const int steps_per_unit = (MODE & 2) ? 2 * ntile : ntile;
  const int my_units = (units - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int total = my_units * steps_per_unit;
  if (threadIdx.x >= 288) {           // MODE 16: idle warps spinning on a never-completing barrier
    if (MODE & 16) {
      uint32_t d = 0; long long n = 0;
      while (!d && n < (1LL << 40)) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(d) : "r"(relay0 + 8 * ST), "r"(0) : "memory");
        ++n;
        if (*(volatile uint32_t*)(sm + ST * STAGE) == 1) break;   // loaders done
      }
    }
    return;
  }
  if (threadIdx.x >= 256) {           // relay warp: waits full(k), arrives relay(k)
    if (threadIdx.x == 256) {
      unsigned acc = 0;
      for (int k = 0; k < total; ++k) {
        const int s = k % ST;
        mwait(full0 + 8 * s, (k / ST) & 1);
        acc += sm[s * STAGE + (k & 1023)];
        marrive(relay0 + 8 * s);
      }
      if (acc == 0x1234567) out[0] = acc;
    }
    return;
  }
  constexpr int CPR = D / 8, RPP = 256 / CPR;
  const int cr = threadIdx.x % CPR, rsub = threadIdx.x / CPR;
  const int b = (MODE & 4) ? bsz : 16;
  auto issue = [&](int k) {
    const int s = k % ST;
    const int u_idx = k / steps_per_unit, i = k % steps_per_unit;
    const int unit = blockIdx.x + u_idx * gridDim.x;
    const int h = unit % HKV, l = (unit / HKV) % L, r = unit / (HKV * L);
    const int tile = (MODE & 2) ? (i < ntile ? i : 2 * ntile - 1 - i) : i;
    const uint32_t stage = su(sm + s * STAGE) + (cr >> 3) * (TILE * 128);
#pragma unroll
    for (int j = 0; j < TILE / RPP; ++j) {
      const int row = RPP * j + rsub, t = tile * TILE + row;
      const int blk = __ldg(tables + r * NB + t / b);
      const uint16_t* src = K + ((((size_t)l * NT + blk) * b + t % b) * HKV + h) * D + cr * 8;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(stage + row * 128 + (((cr & 7) ^ (row & 7)) << 4)), "l"(src) : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full0 + 8 * s) : "memory");
  };
  if (threadIdx.x == 0) *(volatile uint32_t*)(sm + ST * STAGE) = 0;
  for (int k = 0; k < ST && k < total; ++k) issue(k);
  for (int k = 0; k < total; ++k) {
    const int s = k % ST;
    if (MODE & 1) mwait(relay0 + 8 * s, (k / ST) & 1);   // refill only after the relay saw step k
    else mwait(full0 + 8 * s, (k / ST) & 1);
    if (k + ST < total) issue(k + ST);
  }
  if (threadIdx.x == 0) *(volatile uint32_t*)(sm + ST * STAGE) = 1;
}

template <int MODE>
void run(const uint16_t* K, const int* tables, unsigned* out) {
  auto kern = ring<MODE>;
  const int smem = (MODE & 8) ? 210 * 1024 : ST * STAGE + 2048;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    kern<<<148, 352, smem>>>(K, tables, R * L * HKV, 16, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  const double bytes = (double)R * L * HKV * T * D * 2 * ((MODE & 2) ? 2 : 1);
  printf("mode %2d spin=%d (relay=%d 2pass=%d rtdiv=%d bigsmem=%d): %.3f ms  %.1f GB/s smem-fill  (%s)\n", MODE, (MODE >> 4) & 1, MODE & 1, (MODE >> 1) & 1,
         (MODE >> 2) & 1, (MODE >> 3) & 1, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t pool = (size_t)L * NT * 16 * HKV * D * 2;
  uint16_t* K; int* tables; unsigned* out;
  cudaMalloc(&K, pool); cudaMalloc(&out, 4); cudaMemset(K, 1, pool);
  std::vector<int> perm(NT); for (int i = 0; i < NT; ++i) perm[i] = i;
  std::mt19937 g(1); std::shuffle(perm.begin(), perm.end(), g);
  cudaMalloc(&tables, sizeof(int) * R * NB);
  cudaMemcpy(tables, perm.data(), sizeof(int) * R * NB, cudaMemcpyHostToDevice);
  run<15>(K, tables, out); run<16>(K, tables, out); run<31>(K, tables, out);
  return 0;
}
