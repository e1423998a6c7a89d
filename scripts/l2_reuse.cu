// L2 reuse probe for the scoring kernel's K access pattern: 148 CTAs each stream their own slice of a
// [tokens][h_kv=4][256 B] buffer (one head: 256 B rows at 1 KB stride, like a paged K pool) in 32 KB
// tiles, and re-read each tile LAG tiles later. With LAG * 32 KB * 148 well below the L2 size, the
// re-reads should hit L2: run under ncu and compare dram__bytes_read with 1x / 2x the tile bytes.
//   ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum ./l2_reuse
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <int MODE>   // 0: cp.async.cg, 1: ld.global (LDG.128), 2: ld.global.cg
__global__ void __launch_bounds__(256, 1) k(const uint8_t* buf, int tiles, int lag, int head, float* out) {
  if (head < 0) head = blockIdx.x & 3;   // heads vary across CTAs (as units do in the scoring kernel)
  __shared__ __align__(16) uint8_t st[32768];
  const size_t slice = (size_t)tiles * 128 * 1024;   // 128 tokens x 1 KB per tile
  const uint8_t* base = buf + blockIdx.x * slice + head * 256;
  float acc = 0.f;
  // step i: read tile i (if i < tiles), then re-read tile i - lag (if >= 0)
  for (int i = 0; i < tiles + lag; ++i) {
    for (int pass = 0; pass < 2; ++pass) {
      const int t = pass == 0 ? i : i - lag;
      if (t < 0 || t >= tiles) continue;
      const uint8_t* tb = base + (size_t)t * 128 * 1024;
      // 128 rows x 256 B = 2048 x 16 B chunks; 256 threads x 8
      for (int c = threadIdx.x; c < 2048; c += 256) {
        const int row = c >> 4, col = c & 15;
        const uint8_t* src = tb + (size_t)row * 1024 + col * 16;
        if (MODE == 0) {
          cp16((uint32_t)__cvta_generic_to_shared(st + c * 16), src);
        } else if (MODE == 1) {
          const uint4 v = *reinterpret_cast<const uint4*>(src);
          acc += __uint_as_float(v.x ^ v.y ^ v.z ^ v.w);
        } else {
          uint4 v;
          asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src));
          acc += __uint_as_float(v.x ^ v.y ^ v.z ^ v.w);
        }
      }
      if (MODE == 0) { asm volatile("cp.async.wait_all;" ::: "memory"); __syncthreads(); acc += (float)st[threadIdx.x]; }
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const int tiles = 64;                      // 64 x 128 KB per CTA (32 KB read per tile, one head)
  const size_t bytes = (size_t)148 * tiles * 128 * 1024;
  uint8_t* buf;
  float* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  const int lags[] = {1, 4, 8, 16, 32, 64};
  for (int mode = 0; mode < 4; ++mode)
    for (int li = 0; li < 6; ++li) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) k<0><<<148, 256>>>(buf, tiles, lags[li], 0, out);
        if (mode == 1) k<1><<<148, 256>>>(buf, tiles, lags[li], 0, out);
        if (mode == 2) k<2><<<148, 256>>>(buf, tiles, lags[li], 0, out);
        if (mode == 3) k<0><<<148, 256>>>(buf, tiles, lags[li], -1, out);   // cp.async, head = CTA % 4
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      const double uniq = 148.0 * tiles * 32768;
      printf("mode %d lag %2d (reuse distance %6.1f MB): %.3f ms  unique %.1f MB -> %.0f GB/s of unique bytes (%s)\n", mode,
             lags[li], lags[li] * 32768.0 * 148 / 1e6, ms, uniq / 1e6, uniq / (ms * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
