// Replica of the pass-1 epilogue (per-column online log-sum-exp over TMEM logits) in several code
// shapes, to separate the cost of the online-max dependency from the exp2 (MUFU) rate.
//   V0: fixed reference (floor)        V1: linear FMNMX3 chain -> rescale -> exps (kernel r1)
//   V2: tree max -> rescale -> exps     V3: lazy reference: exps use the current reference, the batch
//                                           max (off the MUFU path) only triggers a rare re-base
// EPI = epilogue warps (8: two per TMEM lane quarter, 128 tokens each; 16: four, 64 tokens each).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/p1v scripts/pass1_var.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
#define TMEM_LD16(taddr, v, off) asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
  : "=f"(v[off+0]),"=f"(v[off+1]),"=f"(v[off+2]),"=f"(v[off+3]),"=f"(v[off+4]),"=f"(v[off+5]),"=f"(v[off+6]),"=f"(v[off+7]),"=f"(v[off+8]),"=f"(v[off+9]),"=f"(v[off+10]),"=f"(v[off+11]),"=f"(v[off+12]),"=f"(v[off+13]),"=f"(v[off+14]),"=f"(v[off+15]) : "r"(taddr))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint64_t pk2(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float max3f(float a, float b, float c) { float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }

template <int N>
__device__ __forceinline__ float sum_exp_n(const float* v, float scale, float m) {
  uint64_t acc[4] = {0, 0, 0, 0};
  const uint64_t S2 = pk2(scale, scale), NM2 = pk2(-m, -m);
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const uint64_t arg = fma2(pk2(v[2 * j], v[2 * j + 1]), S2, NM2);
    float a0, a1;
    upk2(arg, a0, a1);
    acc[j & 3] = add2(acc[j & 3], pk2(ex2f(a0), ex2f(a1)));
  }
  const uint64_t s2 = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
  float a, b;
  upk2(s2, a, b);
  return a + b;
}
template <int N>
__device__ __forceinline__ float max_chain(const float* v) {
  float mx = max3f(v[0], v[1], v[2]);
#pragma unroll
  for (int j = 3; j < N - 1; j += 2) mx = max3f(mx, v[j], v[j + 1]);
  return fmaxf(mx, v[N - 1]);
}
template <int N>
__device__ __forceinline__ float max_tree(const float* v) {
  static_assert(N == 32, "");
  float a[11];
#pragma unroll
  for (int j = 0; j < 10; ++j) a[j] = max3f(v[3 * j], v[3 * j + 1], v[3 * j + 2]);
  a[10] = fmaxf(v[30], v[31]);
  const float b0 = max3f(a[0], a[1], a[2]), b1 = max3f(a[3], a[4], a[5]), b2 = max3f(a[6], a[7], a[8]);
  const float b3 = fmaxf(a[9], a[10]);
  return fmaxf(max3f(b0, b1, b2), b3);
}

template <int V, int EPI, int POLL>
__global__ void __launch_bounds__(EPI * 32 + ((POLL == 1 || POLL == 2 || POLL >= 4) ? 256 : 0), 1) k(float* out, int steps, const int4* gsrc) {
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t pbar[2];
  __shared__ volatile int stop;
  extern __shared__ __align__(1024) uint8_t ring[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&pbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;" ::"r"((uint32_t)__cvta_generic_to_shared(&pbar[1])));
  }
  __syncthreads();
  if (POLL >= 4 && warp >= EPI) {
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
    return;
  }
  if ((POLL == 1 || POLL == 2) && warp >= EPI) {
    // warps EPI..EPI+3: pollers (try_wait + nanosleep(100)) on a barrier that never completes;
    // warps EPI+4..EPI+7 (POLL == 2): cp.async streams with a noinc mbarrier arrival per 16 copies
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&pbar[0]);
    const uint32_t b1 = (uint32_t)__cvta_generic_to_shared(&pbar[1]);
    if (warp < EPI + 4) {
      while (!stop) {
        uint32_t d;
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(d) : "r"(b0), "r"(0) : "memory");
        if (!d) __nanosleep(100);
      }
    } else if (POLL == 2) {
      const int lt = threadIdx.x - (EPI + 4) * 32;
      size_t pos = ((size_t)blockIdx.x * 7919 + lt) * 64;
      const size_t gsz = (size_t)1 << 26;
      for (int it = 0; !stop; ++it) {
        for (int kk = 0; kk < 16; ++kk) {
          const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring) + (uint32_t)(((it * 16 + kk) * 128 + lt) % 6144) * 16;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gsrc + (pos % gsz)) : "memory");
          pos += 64 * 16 + 1;
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(b1) : "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      asm volatile("cp.async.wait_all;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
    return;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); asm volatile("bar.sync 1, %0;" ::"r"(EPI * 32)); asm volatile("tcgen05.fence::after_thread_sync;");
  const int q = warp & 3;
  constexpr int TOK = EPI == 8 ? 128 : 64;       // tokens per thread per step
  const int part = warp >> 2;                     // 0..EPI/4-1
  const int half = EPI == 8 ? part : (part & 1);
  const int toff = EPI == 8 ? 0 : (part >> 1) * 64;
  const uint32_t lane_base = slot + ((uint32_t)(q * 32) << 16);
  // fill TMEM with logits in a sane range: value = ((lane*37 + col*11) % 97) * 0.25 - 12
  if (part < 2 || EPI == 16) {
    for (int col = (EPI == 8 ? part * 256 : part * 128); col < (EPI == 8 ? part * 256 + 256 : part * 128 + 128); col += 16) {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(((q * 32 + lane) * 37 % 97 + (col + j) * 11 % 89) * 0.25f - 12.f);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                   ::"r"(lane_base + col), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); asm volatile("bar.sync 1, %0;" ::"r"(EPI * 32)); asm volatile("tcgen05.fence::after_thread_sync;");
  const float scale = 0.1275f;
  float m = -INFINITY, ssum = 0.f;
  constexpr int NB = 32;
  const long long c0 = clock64();
  for (int st = 0; st < steps; ++st) {
    const int a = st & 1;
    if (POLL == 3 || POLL >= 4) asm volatile("bar.sync 2, %0;" ::"r"(EPI * 32) : "memory");
    if (POLL == 6) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (st % 64 == 0) { m = -INFINITY; }        // new unit every 64 steps
    float va[NB], vb[NB];
    const uint32_t tb = lane_base + a * 256 + half * 128 + toff;
    TMEM_LD16(tb, va, 0);
    TMEM_LD16(tb + 16, va, 16);
    auto batch = [&](float* v, float* vn, int bh) {
      tmem_wait_ld();
      if (bh + 1 < TOK / NB) { TMEM_LD16(tb + (bh + 1) * NB, vn, 0); TMEM_LD16(tb + (bh + 1) * NB + 16, vn, 16); }
      else if (POLL == 6) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&pbar[1])) : "memory");
      }
      if (V == 0) {
        ssum += sum_exp_n<NB>(v, scale, 3.0f);
      } else if (V == 1 || V == 2) {
        const float mx = V == 1 ? max_chain<NB>(v) : max_tree<NB>(v);
        const float mn = fmaxf(m, mx * scale);
        const float mref = mn > -INFINITY ? mn : 0.f;
        const float rescale = ex2f(m - mref);
        const float bsum = sum_exp_n<NB>(v, scale, mref);
        ssum = ssum * rescale + bsum;
        m = mn;
      } else {
        const float mx = max_tree<NB>(v) * scale;
        if (mx > m + 64.f) {                       // rare: first batch of a unit / a much larger logit
          const float mref = mx;
          ssum = ssum * ex2f(m - mref) + sum_exp_n<NB>(v, scale, mref);
          m = mref;
        } else {
          ssum += sum_exp_n<NB>(v, scale, m);
        }
      }
    };
    if (POLL == 6) {
      // the kernel's end-of-step release: fence, warp sync, one arrival per warp on an mbarrier
      // (done after the step's last TMEM load, before its math, as in k_score_tc)
    }
    if (TOK / NB == 4) {
#pragma unroll 1
      for (int bh = 0; bh < 4; bh += 2) { batch(va, vb, bh); batch(vb, va, bh + 1); }
    } else {
      batch(va, vb, 0);
      batch(vb, va, 1);
    }
    if (EPI == 16 || part < 2) {}
  }
  if (ssum == 1234.5f) out[0] = ssum + m;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(clock64() - c0);
  if (threadIdx.x == 0) stop = 1;
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int V, int EPI, int POLL>
void run() {
  float* out; cudaMalloc(&out, 8);
  static int4* gsrc = nullptr;
  if (!gsrc) { cudaMalloc(&gsrc, ((size_t)1 << 26) * 16); cudaMemset(gsrc, 0, ((size_t)1 << 26) * 16); }
  cudaFuncSetAttribute(k<V, EPI, POLL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int steps = 4096; float ms = 0;
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(a);
    if (POLL >= 4) {
      cudaFuncSetAttribute(k<V, EPI, POLL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148); cfg.blockDim = dim3(EPI * 32 + 256); cfg.dynamicSmemBytes = 200 * 1024;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = POLL >= 5 ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k<V, EPI, POLL>, out, steps, (const int4*)gsrc);
    } else {
      k<V, EPI, POLL><<<148, EPI * 32 + ((POLL == 1 || POLL == 2) ? 256 : 0), 100 * 1024>>>(out, steps, gsrc);
    }
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  float hc[2]; cudaMemcpy(hc, out, 8, cudaMemcpyDeviceToHost);
  printf("cycles/step %.0f  ", hc[1] / steps);
  printf("pass-1 replica V%d EPI=%2d POLL=%d: %.3f us/step (%s)\n", V, EPI, POLL, ms * 1e3 / steps, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<1, 8, 3>(); run<1, 8, 6>();
  run<3, 8, 3>(); run<3, 8, 6>();
  return 0;
}
