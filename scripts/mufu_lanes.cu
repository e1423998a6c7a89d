// Does MUFU.EX2 throughput depend on the number of active lanes? 8 warps/SM, 2 per SMSP, each
// issuing N independent ex2 per iteration, with 32 / 28 / 16 / 8 active lanes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin_mufu_lanes mufu_lanes.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int ACTIVE>
__global__ void k(float* out, int iters) {
  const int lane = threadIdx.x & 31;
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (i + lane);
  long long t0 = clock64();
  if (lane < ACTIVE) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    }
  }
  __syncwarp();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
}
int main() {
  float* o; cudaMalloc(&o, 8);
  const int iters = 4096;
  auto run = [&](auto kern, int act) {
    kern<<<148, 256>>>(o, iters);   // 8 warps per SM = 2 per SMSP
    kern<<<148, 256>>>(o, iters);
    float c; cudaMemcpy(&c, o + 1, 4, cudaMemcpyDeviceToHost);
    const double per = c / (iters * 16.0);
    printf("active=%2d: %.2f cycles per ex2 warp-instr per SMSP-pair -> %.2f cycles/instr/SMSP (2 warps)\n", act, per, per / 2);
  };
  run(k<32>, 32); run(k<28>, 28); run(k<16>, 16); run(k<8>, 8); run(k<1>, 1);
  return 0;
}
