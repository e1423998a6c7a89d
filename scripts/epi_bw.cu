#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
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
// 2^x on MUFU for most pairs, on the FMA pipe for pairs j % 4 == 3 (25%): balances the two pipes.
template <int J>
__device__ __forceinline__ uint64_t ex2_pair(uint64_t a2) {
  if constexpr ((J & 3) == 3) {
    return ex2_poly2(a2);
  } else {
    float a0, a1;
    upk2(a2, a0, a1);
    return pk2(ex2f(a0), ex2f(a1));
  }
}

// sum_j 2^(v[j]*scale - m) over a 64-value batch, packed
template <int J>
__device__ __forceinline__ void sum_exp_rec(const float* v, uint64_t S2, uint64_t NM2, uint64_t* acc) {
  if constexpr (J < 32) {
    const uint64_t arg = fma2(pk2(v[2 * J], v[2 * J + 1]), S2, NM2);
    acc[J & 3] = add2(acc[J & 3], ex2_pair<J>(arg));
    sum_exp_rec<J + 1>(v, S2, NM2, acc);
  }
}
__device__ __forceinline__ float sum_exp64(const float* v, float scale, float m) {
  uint64_t acc[4] = {0, 0, 0, 0};
  sum_exp_rec<0>(v, pk2(scale, scale), pk2(-m, -m), acc);
  const uint64_t s2 = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
  float a, b;
  upk2(s2, a, b);
  return a + b;
}


__global__ void __launch_bounds__(256, 1) k(float* out, int iters) {
  float v[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) v[j] = -0.37f * ((threadIdx.x * 7 + j * 13) % 50);
  float acc = 0.f, m = 1.0f;
  for (int i = 0; i < iters; ++i) {
    acc += sum_exp64(v, 0.1275f, m);
    m += 1e-7f;
  }
  if (acc == 1234.5f) out[0] = acc;
}
int main() {
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4000; float ms = 0;
  for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k<<<148, 256>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); }
  // per SM: 256 threads x 64 exps per call
  printf("sum_exp64: %.3f ms -> %.3f us per 64-column batch of 256 threads; %.1f exps/clk/SM\n", ms, ms * 1e3 / iters,
         148.0 * 256 * 64 * iters / (ms * 1e-3) / 148 / 1.965e9);
  return 0;
}
