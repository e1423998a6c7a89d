// Host side of the C ABI (include/zipc.h): argument validation, workspace carving, stage
// orchestration on the caller's stream, and the host-buffer e2e variant. No allocation, no
// global state, no stream synchronisation.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"

namespace zpc {
namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

bool desc_ok(const zpc_cache_desc* d, const zpc_params* p) {
  if (!d || !p) return false;
  if (d->num_layers < 1 || d->num_kv_heads < 1 || d->num_q_heads < 1) return false;
  if (d->num_q_heads % d->num_kv_heads) return false;
  if (d->head_dim != 64 && d->head_dim != 128) return false;
  if (d->block_size < 1 || d->num_blocks < 1 || d->num_q_slots < 1 || d->window < 1) return false;
  if (d->dtype != ZPC_BF16 && d->dtype != ZPC_FP32) return false;
  const int G = d->num_q_heads / d->num_kv_heads;
  if ((long long)G * d->window > 256) return false;
  // kernels address a (layer, pool) plane with 32-bit element offsets: per-layer K (or V) element count
  if ((unsigned long long)d->num_blocks * d->block_size * d->num_kv_heads * d->head_dim >= (1ull << 32)) return false;
  if (p->n_max < 2) return false;
  if (p->pool_kernel < 1 || (p->pool_kernel % 2) == 0) return false;
  if (p->max_seq_len < 1 || p->max_seq_len > ZPC_MAX_SEQ_LEN) return false;
  if ((long long)(p->n_max - 1) * d->block_size > (1LL << 30)) return false;
  if (p->flags & ZPC_F_REDUNDANCY) {
    if (!std::isfinite(p->redundancy_lambda) || !std::isfinite(p->redundancy_tau) || !std::isfinite(p->redundancy_p)) return false;
    if (p->redundancy_lambda < 0.f || p->redundancy_tau <= 0.f) return false;
    if (p->redundancy_p < 0.f || p->redundancy_p > 1.f) return false;
    // b <= 32: one warp per block; bf16 b = 48..256 (multiples of 16): the tile kernel
    if (d->block_size > 32 && !(d->dtype == ZPC_BF16 && d->block_size % 16 == 0 && d->block_size <= 256)) return false;
  }
  if (p->flags & ZPC_F_GLOBAL_SCORE) {
    if (!std::isfinite(p->global_alpha) || p->global_alpha < 0.f || p->global_alpha > 1.f) return false;
  }
  if ((p->variant & ~ZPC_V_MASK) != 0 || ((p->variant >> ZPC_V_SELECT_SHIFT) & 3u) == 3u ||
      ((p->variant >> ZPC_V_COMPACT_SHIFT) & 7u) > 4u)
    return false;
  return true;
}

struct LayoutSizes {
  zpc_workspace_layout pub;
  size_t req_err, n_blocks, fresh_off, priv_off, glob, marks, coop_part, coop_cnt, coop_rs, select_keys;
  int32_t coop_cmax;
};

bool compute_layout(const zpc_cache_desc* d, const zpc_params* p, int32_t R, LayoutSizes* o) {
  if (!desc_ok(d, p) || R < 0) return false;
  const size_t units = (size_t)R * d->num_layers * d->num_kv_heads;
  const int G = d->num_q_heads / d->num_kv_heads;
  const int kept_stride = (p->n_max - 1) * d->block_size;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t at = off; off = align_up(off + bytes); return at; };
  memset(o, 0, sizeof(*o));
  o->pub.scores = take(units * p->max_seq_len * sizeof(float));
  o->pub.kept = take(units * kept_stride * sizeof(int32_t));
  o->pub.targets = take((size_t)R * (p->n_max - 1) * sizeof(int32_t));
  o->pub.reserved = take((size_t)R * sizeof(int32_t));
  o->pub.n_prefix = take((size_t)R * sizeof(int32_t));
  o->pub.lse = take(units * G * d->window * sizeof(float));
  o->pub.moves = take(sizeof(unsigned long long));
  o->pub.redundancy = take((p->flags & ZPC_F_REDUNDANCY) ? units * p->max_seq_len * sizeof(float) : 0);
  o->pub.internal = off;
  o->req_err = take((size_t)R * sizeof(int32_t));
  o->n_blocks = take((size_t)R * sizeof(int32_t));
  o->fresh_off = take((size_t)R * sizeof(int32_t));
  o->priv_off = take((size_t)R * sizeof(int32_t));
  o->glob = take(8 * sizeof(int32_t));
  o->marks = take((size_t)d->num_blocks * sizeof(int32_t));
  o->coop_cmax = coop_cmax(p->max_seq_len);
  o->coop_part = take(units * o->coop_cmax * G * d->window * sizeof(float));
  o->coop_cnt = take(units * 2 * sizeof(int32_t));
  o->coop_rs = take((units + 2) * sizeof(int32_t));
  o->select_keys = take(p->max_seq_len > kSelectSmemMaxT ? units * p->max_seq_len * sizeof(uint32_t) : 0);
  o->pub.total_bytes = off;
  o->pub.kept_stride = kept_stride;
  return true;
}

// Builds the kernel-side view of a call. Returns ZPC_OK or a host-detectable error.
int make_call(const zpc_cache_desc* d, const zpc_params* p, const zpc_batch* b, Call* c) {
  LayoutSizes ls;
  if (!b || !compute_layout(d, p, b->num_requests, &ls)) return ZPC_ERR_INVALID_ARG;
  if (!b->status || !b->workspace) return ZPC_ERR_INVALID_ARG;
  if (b->num_requests > 0 && (!b->k_cache || !b->v_cache || !b->q_cache || !b->q_slots || !b->seq_lens ||
                              !b->block_tables || !b->budgets || !b->new_lens || !b->new_num_blocks))
    return ZPC_ERR_INVALID_ARG;
  if (!b->free_stack || !b->free_top || !b->freed_blocks || !b->num_freed) return ZPC_ERR_INVALID_ARG;
  if (b->table_stride < 1 && b->num_requests > 0) return ZPC_ERR_INVALID_ARG;
  if ((p->flags & ZPC_F_PREFIX) && !b->ref_counts) return ZPC_ERR_INVALID_ARG;
  if ((p->flags & ZPC_F_GLOBAL_SCORE) && (!b->global_scores || !b->is_compressed)) return ZPC_ERR_INVALID_ARG;
  if ((p->flags & ZPC_F_POOL_FIRST) && b->num_requests > 0 && !b->is_compressed) return ZPC_ERR_INVALID_ARG;
  if ((p->flags & ZPC_F_LSE_INPUT) && b->num_requests > 0 && !b->window_lse) return ZPC_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(b->workspace) & (kAlign - 1)) != 0) return ZPC_ERR_INVALID_ARG;
  if (b->workspace_bytes < ls.pub.total_bytes) return ZPC_ERR_WORKSPACE;
  const int esz = d->dtype == ZPC_BF16 ? 2 : 4;
  if (b->num_requests > 0 &&
      ((reinterpret_cast<uintptr_t>(b->k_cache) | reinterpret_cast<uintptr_t>(b->v_cache)) & 15))
    return ZPC_ERR_INVALID_ARG;
  (void)esz;
  memset(c, 0, sizeof(*c));
  c->L = d->num_layers; c->h_kv = d->num_kv_heads; c->h_q = d->num_q_heads;
  c->G = d->num_q_heads / d->num_kv_heads; c->d = d->head_dim; c->b = d->block_size;
  c->N_total = d->num_blocks; c->M = d->num_q_slots; c->w = d->window; c->dtype = d->dtype;
  c->n_max = p->n_max; c->pool_kernel = p->pool_kernel; c->max_seq_len = p->max_seq_len; c->flags = p->flags;
  c->variant = p->variant;
  c->R = b->num_requests; c->table_stride = b->table_stride;
  c->free_capacity = b->free_capacity; c->freed_capacity = b->freed_capacity;
  c->k_cache = b->k_cache; c->v_cache = b->v_cache; c->q_cache = b->q_cache;
  c->q_slots = b->q_slots; c->seq_lens = b->seq_lens; c->tables = b->block_tables; c->budgets = b->budgets;
  c->new_lens = b->new_lens; c->new_num_blocks = b->new_num_blocks; c->ref_counts = b->ref_counts;
  c->free_stack = b->free_stack; c->free_top = b->free_top; c->freed = b->freed_blocks;
  c->num_freed = b->num_freed; c->status = b->status;
  char* w = static_cast<char*>(b->workspace);
  c->ws.scores = reinterpret_cast<float*>(w + ls.pub.scores);
  c->ws.kept = reinterpret_cast<int32_t*>(w + ls.pub.kept);
  c->ws.targets = reinterpret_cast<int32_t*>(w + ls.pub.targets);
  c->ws.reserved = reinterpret_cast<int32_t*>(w + ls.pub.reserved);
  c->ws.n_prefix = reinterpret_cast<int32_t*>(w + ls.pub.n_prefix);
  c->ws.lse = reinterpret_cast<float*>(w + ls.pub.lse);
  c->ws.moves = reinterpret_cast<unsigned long long*>(w + ls.pub.moves);
  c->ws.redund = reinterpret_cast<float*>(w + ls.pub.redundancy);
  c->red_lambda = p->redundancy_lambda; c->red_tau = p->redundancy_tau; c->red_p = p->redundancy_p;
  c->global_alpha = p->global_alpha;
  c->f_cache = b->global_scores;
  c->is_compressed = b->is_compressed;
  c->lse_in = (p->flags & ZPC_F_LSE_INPUT) ? b->window_lse : nullptr;
  c->ws.req_err = reinterpret_cast<int32_t*>(w + ls.req_err);
  c->ws.n_blocks = reinterpret_cast<int32_t*>(w + ls.n_blocks);
  c->ws.fresh_off = reinterpret_cast<int32_t*>(w + ls.fresh_off);
  c->ws.priv_off = reinterpret_cast<int32_t*>(w + ls.priv_off);
  c->ws.glob = reinterpret_cast<int32_t*>(w + ls.glob);
  c->ws.marks = reinterpret_cast<int32_t*>(w + ls.marks);
  c->ws.coop_part = reinterpret_cast<float*>(w + ls.coop_part);
  c->ws.coop_cnt = reinterpret_cast<int32_t*>(w + ls.coop_cnt);
  c->ws.coop_rs = reinterpret_cast<int32_t*>(w + ls.coop_rs);
  c->ws.coop_cmax = ls.coop_cmax;
  c->ws.select_keys = reinterpret_cast<uint32_t*>(w + ls.select_keys);
  c->ws.kept_stride = ls.pub.kept_stride;
  return ZPC_OK;
}

inline int cuda_rc(cudaError_t e) { return e == cudaSuccess ? ZPC_OK : ZPC_ERR_CUDA; }

int run_score(const Call& c, cudaStream_t s) {
  if (c.dtype == ZPC_BF16 && !(c.flags & ZPC_F_SCORE_CUDACORE)) {
    bool used = false;
    cudaError_t e = launch_score_coop(c, s, &used);
    if (e != cudaSuccess) return ZPC_ERR_CUDA;
    if (used) return ZPC_OK;
    e = launch_score_res(c, s, &used);
    if (e != cudaSuccess) return ZPC_ERR_CUDA;
    if (used) return ZPC_OK;
    e = launch_score_tc(c, s, &used);
    if (e != cudaSuccess) return ZPC_ERR_CUDA;
    if (used) return ZPC_OK;
  }
  return cuda_rc(launch_score_cudacore(c, s));
}

// ZPC_F_HOST_MAPPED: the host arrays are read / written in place by one kernel per direction (int32 words)
struct HostSeg { const int32_t* src; int32_t* dst; uint32_t words; };
constexpr int kMaxHostSegs = 12;
struct HostSegs { HostSeg s[kMaxHostSegs]; int n; };
__global__ void __launch_bounds__(256) k_host_io(HostSegs g) {
  const HostSeg sg = g.s[blockIdx.y];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < sg.words; i += gridDim.x * blockDim.x)
    sg.dst[i] = sg.src[i];
}
cudaError_t host_io(const HostSegs& g, cudaStream_t s) {
  if (g.n == 0) return cudaSuccess;
  uint32_t mx = 0;
  for (int i = 0; i < g.n; ++i) mx = mx > g.s[i].words ? mx : g.s[i].words;
  const unsigned gx = (unsigned)std::min<uint32_t>(64u, (mx + 255u) / 256u);
  k_host_io<<<dim3(gx > 0 ? gx : 1u, (unsigned)g.n), 256, 0, s>>>(g);
  return cudaGetLastError();
}
void add_seg(HostSegs& g, const void* src, void* dst, size_t bytes) {
  if (bytes == 0 || !src || !dst) return;
  g.s[g.n++] = HostSeg{static_cast<const int32_t*>(src), static_cast<int32_t*>(dst), (uint32_t)(bytes / 4)};
}
}  // namespace
}  // namespace zpc

using namespace zpc;

extern "C" {

int zpc_abi_version(void) { return ZPC_ABI_VERSION; }

size_t zpc_workspace_bytes(const zpc_cache_desc* d, const zpc_params* p, int32_t R) {
  LayoutSizes ls;
  return compute_layout(d, p, R, &ls) ? ls.pub.total_bytes : 0;
}

int zpc_workspace_layout_get(const zpc_cache_desc* d, const zpc_params* p, int32_t R, zpc_workspace_layout* out) {
  LayoutSizes ls;
  if (!out || !compute_layout(d, p, R, &ls)) return ZPC_ERR_INVALID_ARG;
  *out = ls.pub;
  return ZPC_OK;
}

#define ZPC_STAGE(name, body)                                                     \
  int name(const zpc_cache_desc* d, const zpc_params* p, const zpc_batch* b, void* stream) { \
    Call c;                                                                        \
    int rc = make_call(d, p, b, &c);                                               \
    if (rc != ZPC_OK) return rc;                                                   \
    cudaStream_t s = static_cast<cudaStream_t>(stream);                            \
    body                                                                           \
  }

ZPC_STAGE(zpc_plan, {
  if (c.flags & ZPC_F_COUNT_MOVES) cudaMemsetAsync(c.ws.moves, 0, sizeof(unsigned long long), s);
  return cuda_rc(launch_plan(c, s));
})
ZPC_STAGE(zpc_score, { return run_score(c, s); })
ZPC_STAGE(zpc_redundancy, {
  if (!(c.flags & ZPC_F_REDUNDANCY)) return ZPC_OK;
  return cuda_rc(launch_redundancy(c, s));
})
ZPC_STAGE(zpc_select, { return cuda_rc(launch_select(c, s)); })
ZPC_STAGE(zpc_compact, { return cuda_rc(launch_compact(c, s)); })
ZPC_STAGE(zpc_finalize, { return cuda_rc(launch_finalize(c, s)); })
ZPC_STAGE(zpc_compress, {
  if (c.flags & ZPC_F_COUNT_MOVES) cudaMemsetAsync(c.ws.moves, 0, sizeof(unsigned long long), s);
  if ((rc = cuda_rc(launch_plan(c, s))) != ZPC_OK) return rc;
  if ((rc = run_score(c, s)) != ZPC_OK) return rc;
  if ((c.flags & ZPC_F_REDUNDANCY) && (rc = cuda_rc(launch_redundancy(c, s))) != ZPC_OK) return rc;
  if ((rc = cuda_rc(launch_select(c, s))) != ZPC_OK) return rc;
  if ((rc = cuda_rc(launch_compact(c, s))) != ZPC_OK) return rc;
  return cuda_rc(launch_finalize(c, s));
})

size_t zpc_workspace_bytes_host(const zpc_cache_desc* d, const zpc_params* p, int32_t R, int32_t table_stride,
                                int32_t free_capacity, int32_t freed_capacity) {
  LayoutSizes ls;
  if (!compute_layout(d, p, R, &ls)) return 0;
  const size_t units = (size_t)R * d->num_layers * d->num_kv_heads;
  size_t off = ls.pub.total_bytes;
  auto take = [&](size_t bytes) { off = align_up(off + bytes); };
  take((size_t)R * sizeof(int32_t) * 4);                       // q_slots, seq_lens, new_num_blocks, is_compressed
  take((size_t)R * table_stride * sizeof(int32_t));             // tables
  take(units * sizeof(int32_t) * 2);                            // budgets, new_lens
  take((size_t)d->num_blocks * sizeof(int32_t));                // ref counts
  take((size_t)free_capacity * sizeof(int32_t));                // free stack
  take((size_t)freed_capacity * sizeof(int32_t));               // freed
  take(4 * sizeof(int32_t));                                    // free_top, num_freed, status
  return off;
}

int zpc_compress_host(const zpc_cache_desc* d, const zpc_params* p, const zpc_batch* h, void* stream) {
  LayoutSizes ls;
  if (!h || !compute_layout(d, p, h->num_requests, &ls)) return ZPC_ERR_INVALID_ARG;
  const size_t need = zpc_workspace_bytes_host(d, p, h->num_requests, h->table_stride, h->free_capacity,
                                               h->freed_capacity);
  if (!h->workspace || h->workspace_bytes < need) return ZPC_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int R = h->num_requests;
  const size_t units = (size_t)R * d->num_layers * d->num_kv_heads;
  char* base = static_cast<char*>(h->workspace);
  size_t off = ls.pub.total_bytes;      // same carving order as zpc_workspace_bytes_host
  auto take = [&](size_t bytes) { char* at = base + off; off = align_up(off + bytes); return at; };
  int32_t* q_slots = reinterpret_cast<int32_t*>(take((size_t)R * 16));
  int32_t* seq_lens = q_slots + R;
  int32_t* nnb = q_slots + 2 * R;
  int32_t* comp = q_slots + 3 * R;
  int32_t* tables = reinterpret_cast<int32_t*>(take((size_t)R * h->table_stride * 4));
  int32_t* budgets = reinterpret_cast<int32_t*>(take(units * 8));
  int32_t* new_lens = budgets + units;
  int32_t* refs = reinterpret_cast<int32_t*>(take((size_t)d->num_blocks * 4));
  int32_t* stack = reinterpret_cast<int32_t*>(take((size_t)h->free_capacity * 4));
  int32_t* freed = reinterpret_cast<int32_t*>(take((size_t)h->freed_capacity * 4));
  int32_t* small = reinterpret_cast<int32_t*>(take(16));
  const cudaMemcpyKind H2D = cudaMemcpyHostToDevice, D2H = cudaMemcpyDeviceToHost;
  const bool mapped = (p->flags & ZPC_F_HOST_MAPPED) != 0;
  const bool comp_in = (p->flags & (ZPC_F_GLOBAL_SCORE | ZPC_F_POOL_FIRST)) && h->is_compressed;
  if (mapped) {
    HostSegs g;
    g.n = 0;
    if (R) {
      add_seg(g, h->q_slots, q_slots, (size_t)R * 4);
      add_seg(g, h->seq_lens, seq_lens, (size_t)R * 4);
      add_seg(g, h->block_tables, tables, (size_t)R * h->table_stride * 4);
      add_seg(g, h->budgets, budgets, units * 4);
      if (comp_in) add_seg(g, h->is_compressed, comp, (size_t)R * 4);
    }
    if (h->ref_counts) add_seg(g, h->ref_counts, refs, (size_t)d->num_blocks * 4);
    add_seg(g, h->free_stack, stack, (size_t)h->free_capacity * 4);
    add_seg(g, h->free_top, small, 4);
    if (cudaError_t e = host_io(g, s)) return cuda_rc(e);
  } else {
    if (R) {
      cudaMemcpyAsync(q_slots, h->q_slots, (size_t)R * 4, H2D, s);
      cudaMemcpyAsync(seq_lens, h->seq_lens, (size_t)R * 4, H2D, s);
      cudaMemcpyAsync(tables, h->block_tables, (size_t)R * h->table_stride * 4, H2D, s);
      cudaMemcpyAsync(budgets, h->budgets, units * 4, H2D, s);
      if ((p->flags & (ZPC_F_GLOBAL_SCORE | ZPC_F_POOL_FIRST)) && h->is_compressed)
        cudaMemcpyAsync(comp, h->is_compressed, (size_t)R * 4, H2D, s);
    }
    if (h->ref_counts) cudaMemcpyAsync(refs, h->ref_counts, (size_t)d->num_blocks * 4, H2D, s);
    cudaMemcpyAsync(stack, h->free_stack, (size_t)h->free_capacity * 4, H2D, s);
    cudaMemcpyAsync(small, h->free_top, 4, H2D, s);
  }
  zpc_batch dv = *h;
  dv.q_slots = q_slots; dv.seq_lens = seq_lens; dv.block_tables = tables; dv.budgets = budgets;
  dv.new_lens = new_lens; dv.new_num_blocks = nnb; dv.ref_counts = h->ref_counts ? refs : nullptr;
  dv.free_stack = stack; dv.free_top = small; dv.freed_blocks = freed; dv.num_freed = small + 1;
  dv.status = small + 2; dv.workspace = h->workspace; dv.workspace_bytes = ls.pub.total_bytes;
  dv.is_compressed = h->is_compressed ? comp : nullptr;   // global_scores (F), window_lse: device, like K/V/Q
  int rc = zpc_compress(d, p, &dv, stream);
  if (rc != ZPC_OK) return rc;
  if (mapped) {
    HostSegs g;
    g.n = 0;
    if (R) {
      add_seg(g, tables, h->block_tables, (size_t)R * h->table_stride * 4);
      add_seg(g, new_lens, h->new_lens, units * 4);
      add_seg(g, nnb, h->new_num_blocks, (size_t)R * 4);
    }
    if (h->ref_counts) add_seg(g, refs, h->ref_counts, (size_t)d->num_blocks * 4);
    add_seg(g, stack, h->free_stack, (size_t)h->free_capacity * 4);
    add_seg(g, freed, h->freed_blocks, (size_t)h->freed_capacity * 4);
    add_seg(g, small, h->free_top, 4);
    add_seg(g, small + 1, h->num_freed, 4);
    add_seg(g, small + 2, h->status, 4);
    return cuda_rc(host_io(g, s));
  }
  if (R) {
    cudaMemcpyAsync(h->block_tables, tables, (size_t)R * h->table_stride * 4, D2H, s);
    cudaMemcpyAsync(h->new_lens, new_lens, units * 4, D2H, s);
    cudaMemcpyAsync(h->new_num_blocks, nnb, (size_t)R * 4, D2H, s);
  }
  if (h->ref_counts) cudaMemcpyAsync(h->ref_counts, refs, (size_t)d->num_blocks * 4, D2H, s);
  cudaMemcpyAsync(h->free_stack, stack, (size_t)h->free_capacity * 4, D2H, s);
  cudaMemcpyAsync(h->freed_blocks, freed, (size_t)h->freed_capacity * 4, D2H, s);
  cudaMemcpyAsync(h->free_top, small, 4, D2H, s);
  cudaMemcpyAsync(h->num_freed, small + 1, 4, D2H, s);
  cudaMemcpyAsync(h->status, small + 2, 4, D2H, s);
  return cuda_rc(cudaGetLastError());
}

int zpc_score_path(const zpc_cache_desc* d, const zpc_params* p) {
  if (!desc_ok(d, p)) return ZPC_ERR_INVALID_ARG;
  Call c;
  memset(&c, 0, sizeof(c));
  c.L = d->num_layers; c.h_kv = d->num_kv_heads; c.h_q = d->num_q_heads; c.G = d->num_q_heads / d->num_kv_heads;
  c.d = d->head_dim; c.b = d->block_size; c.N_total = d->num_blocks; c.M = d->num_q_slots; c.w = d->window;
  c.dtype = d->dtype; c.n_max = p->n_max; c.pool_kernel = p->pool_kernel; c.max_seq_len = p->max_seq_len;
  c.flags = p->flags; c.variant = p->variant; c.R = 1;
  static const float kDummy = 0.f;                 // only tested against NULL
  c.lse_in = (p->flags & ZPC_F_LSE_INPUT) ? &kDummy : nullptr;
  if (c.dtype == ZPC_BF16 && !(c.flags & ZPC_F_SCORE_CUDACORE)) {
    if (score_coop_applies(c)) return ZPC_PATH_COOP;
    if (score_res_applies(c)) return ZPC_PATH_RESIDENT;
    if (score_tc_applies(c)) return ZPC_PATH_TC;
  }
  return ZPC_PATH_CUDACORE;
}

const char* zpc_status_string(int code) {
  switch (code) {
    case ZPC_OK: return "ok";
    case ZPC_ERR_INVALID_ARG: return "invalid argument";
    case ZPC_ERR_WORKSPACE: return "workspace too small";
    case ZPC_ERR_CUDA: return "CUDA launch error";
    case ZPC_ERR_NOT_TRIGGERED: return "request not triggered (N < N_max)";
    case ZPC_ERR_BAD_TABLE: return "bad block table";
    case ZPC_ERR_BAD_BUDGET: return "budget outside [w, (N_max-1)*b]";
    case ZPC_ERR_NO_FREE_BLOCKS: return "free stack too small for fresh target blocks";
    case ZPC_ERR_SEQ_TOO_LONG: return "seq_len > max_seq_len";
    case ZPC_ERR_BAD_SLOT: return "query slot out of range";
    case ZPC_ERR_CAPACITY: return "freed list or free stack capacity exceeded";
    case ZPC_ERR_NONFINITE: return "non-finite Q or K value (ZPC_F_VALIDATE)";
    default: return "unknown";
  }
}

}  // extern "C"
