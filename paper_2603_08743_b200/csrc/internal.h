// Library-private declarations for libzipc.so (sm_100a). Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "zipc.h"

// Checked builds (-DZPC_CHECKS, scripts/checked_suite.sh): device-side bounds assertions on every gathered /
// scattered pool row, kept index and output position, failing loudly (__trap) -- the stand-in for
// compute-sanitizer memcheck, which this pool does not offer. Compiled out of the product library.
#ifdef ZPC_CHECKS
#include <cstdio>
#define ZPC_CHECK(cond)                                                                                 \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("zpc check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x);                                                                              \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define ZPC_CHECK(cond) do { } while (0)
#endif

namespace zpc {

// Resolved workspace pointers for one call (device addresses).
struct Ws {
  float* scores;           // [R][L][h_kv][max_seq_len]
  int32_t* kept;           // [R][L][h_kv][kept_stride]
  int32_t* targets;        // [R][n_max-1]
  int32_t* reserved;       // [R]
  int32_t* n_prefix;       // [R]
  float* lse;              // [R][L][h_kv][G*w]
  unsigned long long* moves;
  float* redund;           // [R][L][h_kv][max_seq_len] lightning r[t] / T (ZPC_F_REDUNDANCY)
  // internal
  int32_t* req_err;        // [R]
  int32_t* n_blocks;       // [R]
  int32_t* fresh_off;      // [R]  exclusive scan of fresh pops
  int32_t* priv_off;       // [R]  exclusive scan of private frees
  int32_t* glob;           // [8]  0: total_fresh 1: total_priv 2: top_base 3: n_zeroed
  int32_t* marks;          // [N_total] shared blocks driven to 0 (ZPC_F_PREFIX)
  // cooperative score kernel (score_coop.cu): per-chunk partial log2-sum-exp, per-(unit, CTA) arrival
  // counters, the round plan (first unit of each round + the round count)
  float* coop_part;        // [units][coop_cmax][G*w]
  int32_t* coop_cnt;       // [units][2]
  int32_t* coop_rs;        // [units + 2]
  int32_t coop_cmax;       // chunks per unit the part array holds
  uint32_t* select_keys;   // [units][max_seq_len] orderable keys of k_select<true> (max_seq_len > kSelectSmemMaxT)
  int32_t kept_stride;
};

// Flattened view of one call: geometry + pointers. Passed by value to kernels.
struct Call {
  int32_t L, h_kv, h_q, G, d, b, N_total, M, w, dtype;
  int32_t n_max, pool_kernel, max_seq_len;
  uint32_t flags;
  uint32_t debug;      // tuning/bisection switches (ZPC_SCORE_DEBUG, -DZPC_TUNING builds only), else 0
  uint32_t variant;    // zpc_params.variant (ZPC_V_*)
  float red_lambda, red_tau, red_p;   // ZPC_F_REDUNDANCY parameters
  float global_alpha;                 // ZPC_F_GLOBAL_SCORE decay
  int32_t R, table_stride, free_capacity, freed_capacity;
  void* k_cache;
  void* v_cache;
  const void* q_cache;
  const int32_t* q_slots;
  const int32_t* seq_lens;
  int32_t* tables;
  const int32_t* budgets;
  int32_t* new_lens;
  int32_t* new_num_blocks;
  int32_t* ref_counts;
  int32_t* free_stack;
  int32_t* free_top;
  int32_t* freed;
  int32_t* num_freed;
  int32_t* status;
  float* f_cache;                     // ZPC_F_GLOBAL_SCORE: F [L][N_total][b][h_kv]
  const int32_t* is_compressed;       // ZPC_F_GLOBAL_SCORE: [R]
  const float* lse_in;                // ZPC_F_LSE_INPUT: [L][M][w][h_q] natural-log normalisers, else NULL
  Ws ws;
};

// Element offset of row (layer l, physical block blk, slot s, kv head h) in K/V.
__host__ __device__ inline size_t kv_row(const Call& c, int l, int blk, int s, int h) {
  return ((((size_t)l * c.N_total + blk) * c.b + s) * c.h_kv + h) * (size_t)c.d;
}
// Element offset of the query row (layer l, slot j, window row u, query head hq).
__host__ __device__ inline size_t q_row(const Call& c, int l, int slot, int u, int hq) {
  return ((((size_t)l * c.M + slot) * c.w + u) * c.h_q + hq) * (size_t)c.d;
}

// Kernel launchers (return cudaError_t of the launch).
cudaError_t launch_plan(const Call& c, cudaStream_t s);
cudaError_t launch_finalize(const Call& c, cudaStream_t s);
cudaError_t launch_score_cudacore(const Call& c, cudaStream_t s);
cudaError_t launch_score_tc(const Call& c, cudaStream_t s, bool* used);
cudaError_t launch_score_res(const Call& c, cudaStream_t s, bool* used);   // score_res.cu (w = 16, short units)
// which scoring kernel family a call takes (no launch): the same tests the launchers make
bool score_coop_applies(const Call& c);
bool score_res_applies(const Call& c);
bool score_tc_applies(const Call& c);
cudaError_t launch_score_coop(const Call& c, cudaStream_t s, bool* used);
// smallest chunk of the cooperative score kernel (pair-tiles of 256 tokens per chunk): sizes the per-unit
// chunk bound of the workspace partials
constexpr int kCoopChunkTiles = 4;
constexpr int kSelectSmemMaxT = 49152;   // k_select keeps up to this many keys in shared memory
inline int coop_cmax(int max_seq_len) { return ((max_seq_len + 255) / 256 + kCoopChunkTiles - 1) / kCoopChunkTiles; }
cudaError_t launch_select(const Call& c, cudaStream_t s);
cudaError_t launch_compact(const Call& c, cudaStream_t s);
cudaError_t launch_redundancy(const Call& c, cudaStream_t s);
cudaError_t launch_redundancy_tc(const Call& c, cudaStream_t s);   // k_red_umma (redundancy_tc.cu)

// ---- device helpers ----
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float bf16_to_f32(uint16_t v) { return __uint_as_float(((uint32_t)v) << 16); }

}  // namespace zpc
