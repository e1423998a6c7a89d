// Microbenchmark: achievable HBM bandwidth for the paged-K gather of the score kernel
// (one KV head's 2*d-byte rows, 1 KB apart, through a fragmented block table), vs a plain copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu && ./gather_bw
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

constexpr int L = 28, HKV = 4, D = 128, B = 16, R = 64, T = 8192;
constexpr int NB = T / B;            // blocks per request
constexpr int NT = R * NB + 64;      // pool blocks

// one CTA per (unit, chunk of 1024 tokens); each thread loads 16 B chunks; accumulate a checksum
__global__ void gather(const int4* __restrict__ K, const int* __restrict__ tables, unsigned* out, int chunks) {
  const int unit = blockIdx.x / chunks, ch = blockIdx.x % chunks;
  const int h = unit % HKV, l = (unit / HKV) % L, r = unit / (HKV * L);
  const int tok0 = ch * (T / chunks), ntok = T / chunks;
  unsigned acc = 0;
  // 16 threads per row (256 B); blockDim 256 -> 16 rows per pass
  for (int base = 0; base < ntok; base += 16 * 8) {
    int4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = tok0 + base + k * 16 + threadIdx.x / 16;
      const int blk = tables[r * NB + t / B];
      const size_t row = (((size_t)l * NT + blk) * B + t % B) * HKV + h;
      v[k] = K[row * (D * 2 / 16) + threadIdx.x % 16];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void stream(const int4* __restrict__ K, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v = K[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t pool_bytes = (size_t)L * NT * B * HKV * D * 2;
  int4* K; int* tables; unsigned* out;
  cudaMalloc(&K, pool_bytes); cudaMalloc(&out, 4);
  cudaMemset(K, 1, pool_bytes);
  std::vector<int> perm(NT);
  for (int i = 0; i < NT; ++i) perm[i] = i;
  std::mt19937 g(1); std::shuffle(perm.begin(), perm.end(), g);
  cudaMalloc(&tables, sizeof(int) * R * NB);
  cudaMemcpy(tables, perm.data(), sizeof(int) * R * NB, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double head_bytes = (double)R * L * HKV * T * D * 2;   // algorithmic K bytes
  for (int chunks : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      gather<<<R * L * HKV * chunks, 256>>>(K, tables, out, chunks);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("gather chunks=%d: %.3f ms  %.1f GB/s\n", chunks, ms, head_bytes / ms / 1e6);
    }
  }
  const size_t n = pool_bytes / 16;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    stream<<<148 * 8, 512>>>(K, n, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep == 2) printf("stream read: %.3f ms  %.1f GB/s\n", ms, pool_bytes / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
