// a5: in-place compaction of kept K/V rows (Alg. 4), one CTA per unit (r, l, h).
//
// Alg. 4 is a sequential two-pointer sweep; here rank i of the ascending kept list moves
// row kept[i] -> target slot i. Hazard argument: kept[i] >= i, and a destination
// aliases a source only when both are the same logical position of an own target block, i.e.
// i == kept[i] (skipped as an identity move). Ranks are processed in ascending chunks of kChunk
// rows with every read of a chunk completed (CTA barrier) before any write of it; the writes of
// chunk j land on logical positions < (j+1)*kChunk, below every source of chunks > j, so the
// loads of chunk j+1 may be issued before the stores of chunk j (software pipelining).
// Rows move as 16-byte vectors, coalesced along d.
#include "internal.h"

namespace zpc {
namespace {

constexpr int kThreads = 128;
constexpr int kChunk = 16;           // rows per chunk
constexpr int kMaxVecPerRow = 32;    // d*e/16 <= 32 (fp32, d=128)
constexpr int kRegs = kChunk * kMaxVecPerRow / kThreads;   // 8 int4 per tensor per thread

struct Chunk {
  int4 k[kRegs], v[kRegs];
  uint32_t dst[kRegs];               // destination vector index within the layer-head plane, ~0u = none
};

__device__ __forceinline__ void load_chunk(const Call& c, Chunk& ch, int base, int ell, int vpr, const int32_t* kept,
                                           const int32_t* table, const int32_t* tg, const int4* K, const int4* V,
                                           size_t plane, int esz) {
  const int rows = min(kChunk, ell - base);
  const int nvec = rows * vpr;
#pragma unroll
  for (int k = 0; k < kRegs; ++k) {
    const int v = threadIdx.x + k * kThreads;
    ch.dst[k] = ~0u;
    if (v < nvec) {
      const int i = base + v / vpr, e = v % vpr;
      const int t = kept[i];
      const int sblk = table[t / c.b], dblk = tg[i / c.b];
      // vector index relative to (layer, head) plane: ((blk*b + slot)*h_kv)*vpr + e
      const uint32_t src = (uint32_t)(((size_t)sblk * c.b + t % c.b) * c.h_kv * vpr + e);
      const uint32_t d = (uint32_t)(((size_t)dblk * c.b + i % c.b) * c.h_kv * vpr + e);
      if (src != d) {
        ch.k[k] = K[plane + src];
        ch.v[k] = V[plane + src];
        ch.dst[k] = d;
      }
    }
  }
  (void)esz;
}

__global__ void __launch_bounds__(kThreads, 6) k_compact(Call c) {
  if (*c.status != ZPC_OK) return;
  const int unit = blockIdx.x;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int ell = c.new_lens[unit];
  const int nm1 = c.n_max - 1;
  const int32_t* kept = c.ws.kept + (size_t)unit * c.ws.kept_stride;
  const int32_t* tg = c.ws.targets + (size_t)r * nm1;
  const int32_t* table = c.tables + (size_t)r * c.table_stride;
  const int esz = c.dtype == ZPC_BF16 ? 2 : 4;
  const int vpr = c.d * esz / 16;               // 16-byte vectors per row
  const int4* K = reinterpret_cast<const int4*>(c.k_cache);
  const int4* V = reinterpret_cast<const int4*>(c.v_cache);
  int4* Kw = reinterpret_cast<int4*>(c.k_cache);
  int4* Vw = reinterpret_cast<int4*>(c.v_cache);
  // start of the (layer l, head h) plane in vectors; per-row offsets are 32-bit within a layer
  const size_t plane = (size_t)l * c.N_total * c.b * c.h_kv * vpr + (size_t)h * vpr;
  unsigned moved = 0;

  Chunk cur, nxt;
  if (ell > 0) load_chunk(c, cur, 0, ell, vpr, kept, table, tg, K, V, plane, esz);
  for (int base = 0; base < ell; base += kChunk) {
    __syncthreads();   // every read of chunk `base` has returned before any write of it
    const bool more = base + kChunk < ell;
    if (more) load_chunk(c, nxt, base + kChunk, ell, vpr, kept, table, tg, K, V, plane, esz);
#pragma unroll
    for (int k = 0; k < kRegs; ++k) {
      if (cur.dst[k] != ~0u) {
        Kw[plane + cur.dst[k]] = cur.k[k];
        Vw[plane + cur.dst[k]] = cur.v[k];
        moved += ((threadIdx.x + k * kThreads) % vpr) == 0;
      }
    }
    if (more) cur = nxt;
  }
  if (c.flags & ZPC_F_COUNT_MOVES) {
    for (int o = 16; o; o >>= 1) moved += __shfl_xor_sync(0xffffffffu, moved, o);
    if ((threadIdx.x & 31) == 0 && moved) atomicAdd(c.ws.moves, (unsigned long long)moved);
  }
}

}  // namespace

cudaError_t launch_compact(const Call& c, cudaStream_t s) {
  const int units = c.R * c.L * c.h_kv;
  if (units == 0) return cudaSuccess;
  k_compact<<<units, kThreads, 0, s>>>(c);
  return cudaGetLastError();
}

}  // namespace zpc
