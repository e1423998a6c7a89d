// Microbenchmark of smem-ring loader designs for the paged K gather (1 CTA/SM, 3-4 x 32 KB stages,
// a consumer warp that only waits/releases). Variants: cp.async+mbarrier(noinc), LDG->STS.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int L = 28, HKV = 4, D = 128, B = 16, R = 64, T = 8192;
constexpr int NB = T / B, NT = R * NB + 64, TILE = 128, STAGE = TILE * D * 2;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint32_t b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n)); }
__device__ __forceinline__ void marrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void mwait(uint32_t b, uint32_t ph) {
  uint32_t d = 0;
  while (!d) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(d) : "r"(b), "r"(ph) : "memory");
}

template <int NLD, int ST, int MODE>   // MODE 0: cp.async noinc; 1: LDG->STS (8 int4 batches)
__global__ void __launch_bounds__(NLD + 32, 1) ring(const uint16_t* K, const int* tables, int units, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + ST * STAGE);
  const uint32_t full0 = su(bars), empty0 = su(bars + ST);
  if (threadIdx.x == 0) { for (int s = 0; s < ST; ++s) { minit(full0 + 8 * s, NLD); minit(empty0 + 8 * s, 1); } }
  __syncthreads();
  const int ntile = T / TILE;
  if (threadIdx.x >= NLD) {          // consumer warp
    if (threadIdx.x == NLD) {
      int k = 0; unsigned acc = 0;
      for (int unit = blockIdx.x; unit < units; unit += gridDim.x)
        for (int i = 0; i < ntile; ++i, ++k) {
          const int s = k % ST;
          mwait(full0 + 8 * s, (k / ST) & 1);
          acc += sm[s * STAGE + (i & 1023)];
          marrive(empty0 + 8 * s);
        }
      if (acc == 0x1234567) out[0] = acc;
    }
    return;
  }
  constexpr int CPR = D / 8, RPP = NLD / CPR;
  const int cr = threadIdx.x % CPR, rsub = threadIdx.x / CPR;
  int k = 0;
  for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const int h = unit % HKV, l = (unit / HKV) % L, r = unit / (HKV * L);
    for (int i = 0; i < ntile; ++i, ++k) {
      const int s = k % ST;
      mwait(empty0 + 8 * s, ((k / ST) & 1) ^ 1);
      const uint32_t stage = su(sm + s * STAGE) + (cr >> 3) * (TILE * 128);
      if (MODE == 0) {
#pragma unroll 8
        for (int j = 0; j < TILE / RPP; ++j) {
          const int row = RPP * j + rsub, t = i * TILE + row;
          const int blk = __ldg(tables + r * NB + t / B);
          const uint16_t* src = K + ((((size_t)l * NT + blk) * B + t % B) * HKV + h) * D + cr * 8;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(stage + row * 128 + (((cr & 7) ^ (row & 7)) << 4)), "l"(src) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full0 + 8 * s) : "memory");
      } else {
        for (int j0 = 0; j0 < TILE / RPP; j0 += 8) {
          int4 v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int row = RPP * (j0 + j) + rsub, t = i * TILE + row;
            const int blk = __ldg(tables + r * NB + t / B);
            v[j] = *reinterpret_cast<const int4*>(K + ((((size_t)l * NT + blk) * B + t % B) * HKV + h) * D + cr * 8);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int row = RPP * (j0 + j) + rsub;
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(stage + row * 128 + (((cr & 7) ^ (row & 7)) << 4)), "r"(v[j].x), "r"(v[j].y), "r"(v[j].z), "r"(v[j].w) : "memory");
          }
        }
        marrive(full0 + 8 * s);
      }
    }
  }
}

template <int NLD, int ST, int MODE>
void run(const uint16_t* K, const int* tables, unsigned* out, const char* name) {
  auto kern = ring<NLD, ST, MODE>;
  const int smem = ST * STAGE + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    kern<<<148, NLD + 32, smem>>>(K, tables, R * L * HKV, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  const double bytes = (double)R * L * HKV * T * D * 2;
  printf("%-28s NLD=%3d ST=%d: %.3f ms %.1f GB/s  (%s)\n", name, NLD, ST, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t pool = (size_t)L * NT * B * HKV * D * 2;
  uint16_t* K; int* tables; unsigned* out;
  cudaMalloc(&K, pool); cudaMalloc(&out, 4); cudaMemset(K, 1, pool);
  std::vector<int> perm(NT); for (int i = 0; i < NT; ++i) perm[i] = i;
  std::mt19937 g(1); std::shuffle(perm.begin(), perm.end(), g);
  cudaMalloc(&tables, sizeof(int) * R * NB);
  cudaMemcpy(tables, perm.data(), sizeof(int) * R * NB, cudaMemcpyHostToDevice);
  run<64, 3, 0>(K, tables, out, "cp.async noinc");
  run<128, 3, 0>(K, tables, out, "cp.async noinc");
  run<256, 3, 0>(K, tables, out, "cp.async noinc");
  run<128, 6, 0>(K, tables, out, "cp.async noinc");
  run<64, 3, 1>(K, tables, out, "ldg->sts");
  run<128, 3, 1>(K, tables, out, "ldg->sts");
  run<256, 3, 1>(K, tables, out, "ldg->sts");
  run<256, 6, 1>(K, tables, out, "ldg->sts");
  return 0;
}
