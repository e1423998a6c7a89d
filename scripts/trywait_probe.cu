// How long one mbarrier.try_wait (no suspend hint) on a phase that never completes takes on this GPU:
// calibrates the poll-count hang detector of mbar_wait_lean (tc_util.h).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o trywait_probe scripts/trywait_probe.cu && ./trywait_probe
#include <cstdio>
#include <cstdint>
__global__ void probe(unsigned long long* out, int polls, int hint) {
  __shared__ uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(2));
  __syncthreads();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint32_t done = 0;
  for (int i = 0; i < polls; ++i) {
    if (hint)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(b), "r"(0u), "r"(1000000u) : "memory");
    else
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(b), "r"(0u) : "memory");
    if (done) break;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = done; }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  for (int hint = 0; hint < 2; ++hint) {
    const int polls = 20000;
    probe<<<1, 32>>>(d, polls, hint);
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("hint %d: %d polls in %llu ns -> %.1f ns per poll (done %llu)\n", hint, polls, h[0], (double)h[0] / polls, h[1]);
  }
  return 0;
}
