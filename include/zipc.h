/*
 * zipc.h — C ABI of the B200-native compression step of Compressed PagedAttention
 * (Zipage, arXiv 2603.08743). Library: paper_2603_08743_b200/lib/libzipc.so (sm_100a).
 *
 * What one call computes (PAPER.md = /root/reference/PAPER.md):
 *   For every request r flagged for compression, every layer l and KV head h (a "unit"):
 *   a0 plan      trigger check N >= N_max (§4.1); prefix-aware target blocks
 *                (§4.5); fresh blocks popped from the free stack.
 *   a1 score     logits q.k/sqrt(d) of the last w window queries against every cached key,
 *                read through the block table, causal in absolute positions (Alg. 1,
 *                PAPER.md:369-405).
 *   a2           softmax over each window row, max over the GQA group, mean over the window
 *                  ->  S[t], fp32.
 *   a3 select    MaxPool1D along the sequence, window pinned to +inf
 *                (PAPER.md:85, :591),
 *   a4           keep the top min(T, budget) tokens per head, ties -> later position,
 *                emitted in ascending order.
 *   a5 compact   move kept K/V rows, in order, into the target blocks (Alg. 4).
 *   a6 finalize  new table = targets ++ [reserved]; freed list; ref counts; free-stack push
 *                (PAPER.md:22, :64, :138).
 *   The readings taken where the paper is silent or garbled are DESIGN.md §Readings R1..R17.
 *
 * Conventions for every entry point:
 *   - All array pointers are caller-owned DEVICE memory unless the name says _host.
 *     The library allocates nothing, keeps no mutable global state (the only process-wide value is
 *     the resolved cuTensorMapEncodeTiled driver entry point, written once, read-only after) and
 *     never synchronises the stream; it reads no environment variables.
 *     Outputs are valid after the caller synchronises `stream` (a cudaStream_t; NULL = legacy).
 *   - Host-detectable errors (bad descriptor/params, workspace too small) return a negative
 *     ZPC_ERR_* and enqueue NOTHING.
 *   - Device-detected errors are written to *status (device int32) by the plan stage; every
 *     later stage reads *status at entry and returns without touching memory if it is non-zero.
 *     All-or-nothing: plan checks everything before any mutation.
 *   - Determinism: outputs are bit-identical run to run and independent of how requests are
 *     sharded across GPUs (all per-request quantities; free-list order is defined below).
 *   - Concurrency: two calls may run on different streams only if they share no allocator
 *     (free stack / ref counts), no workspace and no request.
 */
#ifndef ZIPC_H_
#define ZIPC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZPC_ABI_VERSION 6

/* ---- return / status codes ---- */
#define ZPC_OK                  0
#define ZPC_ERR_INVALID_ARG    -1   /* bad descriptor/params: even pool_kernel, w<1, n_max<2,
                                       unsupported head_dim/dtype, h_q not a multiple of h_kv,
                                       G*w > 256, max_seq_len above the select limit, NULL pointer,
                                       a per-layer pool of >= 2^32 elements (N_total*b*h_kv*d; the
                                       kernels use 32-bit offsets inside a layer), unknown variant bits,
                                       ZPC_F_REDUNDANCY with lambda < 0, tau <= 0, p outside [0,1],
                                       a non-finite value, or block_size > 32 unless bf16 with
                                       block_size a multiple of 16 up to 256, ZPC_F_GLOBAL_SCORE
                                       with alpha outside [0,1] or a NULL global_scores /
                                       is_compressed, ZPC_F_LSE_INPUT with a NULL window_lse */
#define ZPC_ERR_WORKSPACE      -2   /* workspace_bytes < zpc_workspace_bytes(...) */
#define ZPC_ERR_CUDA           -3   /* a launch failed (cudaGetLastError) */
#define ZPC_ERR_NOT_TRIGGERED -10   /* device: N = ceil(T/b) < N_max */
#define ZPC_ERR_BAD_TABLE     -11   /* device: N > table_stride, block id out of [0,N_total),
                                       duplicate id (ZPC_F_VALIDATE), or a shared block
                                       (ref > 1) after a private one (ZPC_F_PREFIX) */
#define ZPC_ERR_BAD_BUDGET    -12   /* device: budget outside [w, (N_max-1)*b] */
#define ZPC_ERR_NO_FREE_BLOCKS -13  /* device: free stack holds fewer blocks than the fresh
                                       targets/reserved blocks the plan needs */
#define ZPC_ERR_SEQ_TOO_LONG  -14   /* device: seq_len > params.max_seq_len */
#define ZPC_ERR_BAD_SLOT      -15   /* device: q_slot outside [0, M) */
#define ZPC_ERR_CAPACITY      -16   /* device: freed list or free stack would overflow */
#define ZPC_ERR_NONFINITE     -17   /* device (ZPC_F_VALIDATE): a Q or K element the call reads is Inf/NaN */
/* When several requests fail, *status is the error of the lowest-index failing request
 * (its first failing check in the order SLOT, SEQ_TOO_LONG, TABLE(stride), NOT_TRIGGERED,
 * TABLE(range), TABLE(dup), TABLE(prefix run), BUDGET); batch-level checks come after. */

/* ---- element type of K, V and Q (one type for all three) ---- */
#define ZPC_BF16 0
#define ZPC_FP32 1

/* ---- flags ---- */
#define ZPC_F_PREFIX      1u  /* use ref_counts: leading blocks with ref > 1 are shared (§4.5) */
#define ZPC_F_VALIDATE    2u  /* also reject duplicate block ids inside a table (ZPC_ERR_BAD_TABLE) and any
                                 non-finite Q / K element the call reads (ZPC_ERR_NONFINITE; reads every
                                 K row of the call once more) */
#define ZPC_F_COUNT_MOVES 4u  /* count moved rows into the workspace counter (bytes accounting) */
#define ZPC_F_SCORE_CUDACORE 8u /* force the CUDA-core scoring kernel even for bf16 (testing) */
#define ZPC_F_REDUNDANCY 16u  /* NEXT-1: lightning redundancy score (§C.7) with the
                                 temperature softmax (§C.8) folded into the selection
                                 score after pooling: S = MaxPool(S) - lambda * softmax(r / tau)
                                 (PAPER.md:506). Uses params.redundancy_*; adds a workspace region. */
#define ZPC_F_GLOBAL_SCORE 32u /* NEXT-2: global score, Alg. 2 (§C.3): per block of a
                                 request, F <- S when is_compressed[r] == 0; otherwise S <- max(alpha F,
                                 S) on the logical blocks < N_max-1 (the previous targets), F <- S;
                                 pooling etc. then use the updated S, and compaction moves each kept
                                 row's F with its K/V. Needs batch.global_scores and
                                 batch.is_compressed; params.global_alpha. */
#define ZPC_F_LSE_INPUT 64u   /* NEXT-4: single-pass scoring. batch.window_lse supplies, per layer, query
                                 slot, window row u and query head, the softmax normaliser
                                 LSE = log sum_{t <= T-w+u} exp(q.k_t / sqrt(d)) (natural log) that the
                                 decode attention of position T-w+u already computed (it attends over
                                 exactly the keys 0..T-w+u). a2 then needs one pass over K instead of
                                 two: S[t] = (1/w) sum_u max_g exp(q.k_t/sqrt(d) - LSE[u][g])
                                 (PAPER.md:409-411 with the normaliser given). Results equal the
                                 two-pass ones when the input is the exact normaliser. */

#define ZPC_F_POOL_FIRST 128u /* MaxPool1D only at a request's FIRST compression (pooling at
                                 every step hurts Qwen3-8B; the paper pools at the first compression only):
                                 requests with is_compressed[r] != 0 select on the unpooled score. Needs
                                 batch.is_compressed (as ZPC_F_GLOBAL_SCORE does). */

#define ZPC_F_HOST_MAPPED 256u /* zpc_compress_host only: every host array of the batch is device-accessible at its
                                 host address (page-locked with cudaHostAlloc / cudaHostRegister on a unified-
                                 address system). The call then stages the inputs with ONE gather kernel and
                                 returns the outputs with ONE scatter kernel that read / write the host arrays
                                 directly, instead of one copy per array (a small call is otherwise bound by ~17
                                 copy latencies). Pageable host memory with this flag faults. Ignored elsewhere. */

/* Pool geometry: K, V [L][N_total][b][h_kv][d], Q [L][M][w][h_q][d].
 * Q row u of slot j holds the query of position T-w+u of the request bound to slot j (R3). */
typedef struct {
  int32_t num_layers;    /* L */
  int32_t num_kv_heads;  /* h_kv */
  int32_t num_q_heads;   /* h_q, a multiple of h_kv; query head i uses KV head i / (h_q/h_kv) (R5) */
  int32_t head_dim;      /* d: 64 or 128 */
  int32_t block_size;    /* b >= 1 */
  int32_t num_blocks;    /* N_total */
  int32_t num_q_slots;   /* M */
  int32_t window;        /* w >= 1 (may exceed b) */
  int32_t dtype;         /* ZPC_BF16 or ZPC_FP32 */
} zpc_cache_desc;

typedef struct {
  int32_t n_max;         /* N_max >= 2: blocks per request after compression */
  int32_t pool_kernel;   /* 1 = no pooling; odd >= 3 = MaxPool1D width, stride 1, same length (R6) */
  int32_t max_seq_len;   /* host bound on seq_lens: sizes the workspace and grids (<= ZPC_MAX_SEQ_LEN) */
  uint32_t flags;        /* ZPC_F_* */
  /* ZPC_F_REDUNDANCY only (ignored otherwise; all finite):
   *   redundancy_lambda  lambda >= 0, weight of R in S - lambda*R (PAPER.md:506; 0.2 recommended, :718)
   *   redundancy_tau     tau > 0, temperature of the softmax over the sequence (0.4)
   *   redundancy_p       p in [0, 1], similarity threshold: per column of a block's cosine matrix
   *                      the last (newest-row) entry strictly above p is zeroed (
   *                      the paper gives no value) */
  float redundancy_lambda;
  float redundancy_tau;
  float redundancy_p;
  /* ZPC_F_GLOBAL_SCORE only: decay alpha in [0, 1] (PAPER.md:441; 0.8 recommended, :718) */
  float global_alpha;
  /* Kernel-variant overrides for tests and A/B timing (ZPC_V_*; 0 = automatic choice). Every variant
   * computes the same result; only the launch configuration differs. */
  uint32_t variant;
} zpc_params;

/* ---- zpc_params.variant ---- */
#define ZPC_V_SCORE_SERIAL   1u        /* two-pass tcgen05 scoring: the per-unit serial kernel (k_score_tc)
                                          instead of the cooperative / overlapped ones */
#define ZPC_V_SELECT_SHIFT   4         /* bits 4..5: 0 auto, 1 k_select, 2 k_select_reg (T <= 32K) */
#define ZPC_V_COMPACT_SHIFT  8         /* bits 8..10: 0 auto, 1..4 = k_compact CTA width 128/256/512/1024 */
#define ZPC_V_RED_MMASYNC    (1u << 12) /* ZPC_F_REDUNDANCY, bf16 b = 32..256: the mma.sync block-Gram kernel
                                          (k_red_tile) instead of the tcgen05 one (k_red_umma) */
#define ZPC_V_MASK           0x1733u

#define ZPC_MAX_SEQ_LEN 262144  /* units up to 48K tokens select from shared memory, longer ones from a
                                   workspace key region (max_seq_len x 4 bytes per unit, sized by the
                                   workspace queries) */

/* Everything one call touches. Pointers are device memory. Layouts:
 *   q_slots      int32 [R]                 query slot of each request
 *   seq_lens     int32 [R]                 T_r; N_r = ceil(T_r / b) blocks are in use
 *   block_tables int32 [R][table_stride]   in/out: first N_max entries rewritten
 *   budgets      int32 [R][L][h_kv]        per-head budget, w <= budget <= (N_max-1)*b
 *   new_lens     int32 [R][L][h_kv]  out   kept entries per head = min(T_r, budget) (R8)
 *   new_num_blocks int32 [R]         out   = N_max
 *   ref_counts   int32 [N_total] in/out    or NULL (then ZPC_F_PREFIX must be clear)
 *   free_stack   int32 [free_capacity]     valid entries [0, *free_top); pop = stack[top-1]
 *   freed_blocks int32 [freed_capacity] out, *num_freed out:
 *                private blocks that are neither targets nor reserved, ascending logical
 *                index, requests in input order; then shared blocks this call drove to ref 0,
 *                ascending id. They are also pushed onto the free stack in that order.
 *   status       int32 [1] out             ZPC_OK or a device ZPC_ERR_*
 */
typedef struct {
  void* k_cache;
  void* v_cache;
  const void* q_cache;
  int32_t num_requests;
  const int32_t* q_slots;
  const int32_t* seq_lens;
  int32_t* block_tables;
  int32_t table_stride;
  const int32_t* budgets;
  int32_t* new_lens;
  int32_t* new_num_blocks;
  int32_t* ref_counts;
  int32_t* free_stack;
  int32_t* free_top;
  int32_t free_capacity;
  int32_t* freed_blocks;
  int32_t* num_freed;
  int32_t freed_capacity;
  void* workspace;          /* device scratch, >= zpc_workspace_bytes(...), 256-B aligned */
  size_t workspace_bytes;
  int32_t* status;
  /* ZPC_F_GLOBAL_SCORE only (else ignored, may be NULL):
   *   global_scores  dev fp32 [L][N_total][b][h_kv], in/out: F, the global-score pool
   * ZPC_F_GLOBAL_SCORE or ZPC_F_POOL_FIRST:
   *   is_compressed  dev int32 [R], 0 or 1: the request was compressed before (Alg. 2 line 3) */
  float* global_scores;
  const int32_t* is_compressed;
  /* ZPC_F_LSE_INPUT only (else ignored, may be NULL):
   *   window_lse  dev fp32 [L][M][w][h_q], natural log, laid out like the Q cache without d: entry
   *               (l, j, u, i) is the log-sum-exp of query head i of window row u of slot j over keys
   *               0..T-w+u, logits scaled by 1/sqrt(d). Must be finite. Read only. */
  const float* window_lse;
} zpc_batch;

/* Where intermediate results live inside the workspace (byte offsets; all 256-B aligned). */
typedef struct {
  size_t total_bytes;
  size_t scores;     /* fp32 [R][L][h_kv][max_seq_len]: S before pooling/pinning (a2 output) */
  size_t kept;       /* int32 [R][L][h_kv][kept_stride]: ascending kept positions (a4 output) */
  size_t targets;    /* int32 [R][N_max-1]: physical target block of each rank/b (a0 output) */
  size_t reserved;   /* int32 [R] */
  size_t n_prefix;   /* int32 [R] */
  size_t lse;        /* fp32 [R][L][h_kv][G*w]: log2-domain log-sum-exp per window row/head */
  size_t moves;      /* unsigned long long [1]: rows moved (ZPC_F_COUNT_MOVES) */
  size_t redundancy; /* fp32 [R][L][h_kv][max_seq_len]: lightning row sums r[t] / T before the
                        softmax (ZPC_F_REDUNDANCY; a zero-size region otherwise) */
  size_t internal;   /* library-private scratch */
  int32_t kept_stride;   /* (N_max-1)*b */
} zpc_workspace_layout;

/* Workspace size for R requests; 0 if the descriptor/params are invalid. */
size_t zpc_workspace_bytes(const zpc_cache_desc* desc, const zpc_params* params, int32_t num_requests);
int zpc_workspace_layout_get(const zpc_cache_desc* desc, const zpc_params* params, int32_t num_requests,
                             zpc_workspace_layout* out);

/* The whole step a0..a6, stream-ordered, no host sync. */
int zpc_compress(const zpc_cache_desc* desc, const zpc_params* params, const zpc_batch* batch, void* stream);

/* Stage entry points (same conventions; each consumes the previous stage's workspace output).
 * zpc_plan writes *status, targets/reserved/n_prefix and the internal scan; it mutates nothing
 * outside the workspace and *status. zpc_score writes S and LSE. zpc_select writes kept and
 * new_lens (with ZPC_F_REDUNDANCY it reads the `redundancy` region written by zpc_redundancy; with
 * ZPC_F_GLOBAL_SCORE it applies Alg. 2 first: updates F and overwrites S with the global score).
 * zpc_compact moves K/V rows (and F rows with ZPC_F_GLOBAL_SCORE). zpc_finalize rewrites tables, ref counts, freed list,
 * free stack and top, new_num_blocks. */
int zpc_plan(const zpc_cache_desc* desc, const zpc_params* params, const zpc_batch* batch, void* stream);
int zpc_score(const zpc_cache_desc* desc, const zpc_params* params, const zpc_batch* batch, void* stream);
/* NEXT-1 (ZPC_F_REDUNDANCY): per unit and block of b tokens, the b x b cosine similarity of the
 * block's keys (diagonal zeroed, per column the last entry > p zeroed), row sums / T into the
 * workspace `redundancy` region; slots >= T take no part, a zero-norm key has cosine 0.
 * zpc_compress runs it between score and select; as a stage it is a no-op without the flag.
 * zpc_select then folds lambda * softmax(r / tau) in. */
int zpc_redundancy(const zpc_cache_desc* desc, const zpc_params* params, const zpc_batch* batch, void* stream);
int zpc_select(const zpc_cache_desc* desc, const zpc_params* params, const zpc_batch* batch, void* stream);
int zpc_compact(const zpc_cache_desc* desc, const zpc_params* params, const zpc_batch* batch, void* stream);
int zpc_finalize(const zpc_cache_desc* desc, const zpc_params* params, const zpc_batch* batch, void* stream);

/* End-to-end variant for host-resident bookkeeping (the e2e benchmark path): `host` holds the
 * same fields, but q_slots, seq_lens, block_tables, budgets, new_lens, new_num_blocks,
 * ref_counts, free_stack, free_top, freed_blocks, num_freed, status and is_compressed point to HOST
 * memory (pinned for async copies); k_cache, v_cache, q_cache, global_scores and workspace are
 * device memory.
 * The call stages the host inputs into the workspace (H2D), runs zpc_compress, and copies every
 * output back (D2H), all on `stream` (per-array copies, or one gather / one scatter kernel with
 * ZPC_F_HOST_MAPPED). Host buffers must stay alive until the stream is synced.
 * Workspace must be >= zpc_workspace_bytes_host(...). */
size_t zpc_workspace_bytes_host(const zpc_cache_desc* desc, const zpc_params* params, int32_t num_requests,
                                int32_t table_stride, int32_t free_capacity, int32_t freed_capacity);
int zpc_compress_host(const zpc_cache_desc* desc, const zpc_params* params, const zpc_batch* host, void* stream);

/* Which scoring kernel family (a1 + a2) a call with this descriptor and these params runs (no launch, no
 * device access). PAPER.md:369-411 defines what every family computes; they differ only in how:
 *   ZPC_PATH_COOP      tcgen05, cooperative CTA pairs, two passes (bf16, w = 32, G in {5, 7, 8})
 *   ZPC_PATH_RESIDENT  tcgen05, logits resident in TMEM, one MMA pass (bf16, w = 16, G = 4, d = 128,
 *                      max_seq_len <= 4096: the paper's operating point)
 *   ZPC_PATH_TC        tcgen05, per-unit kernels (bf16, w = 32 with G = 1..8 or w = 16 with G in {4, 8};
 *                      single-pass ZPC_F_LSE_INPUT calls; ZPC_V_SCORE_SERIAL)
 *   ZPC_PATH_CUDACORE  FFMA kernels (fp32, other w or G, b < 5, or ZPC_F_SCORE_CUDACORE)
 * Returns one of these, or ZPC_ERR_INVALID_ARG for a descriptor zpc_compress would reject. */
#define ZPC_PATH_COOP      1
#define ZPC_PATH_RESIDENT  2
#define ZPC_PATH_TC        3
#define ZPC_PATH_CUDACORE  4
int zpc_score_path(const zpc_cache_desc* desc, const zpc_params* params);

const char* zpc_status_string(int code);
int zpc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ZIPC_H_ */
