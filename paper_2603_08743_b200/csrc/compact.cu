// a5: in-place compaction of kept K/V rows (Alg. 4), one CTA per unit (r, l, h).
//
// Alg. 4 is a sequential two-pointer sweep; here rank i of the ascending kept list moves
// row kept[i] -> target slot i. Hazard argument: kept[i] >= i, and a
// destination aliases a source only when both are the same logical position of an own target
// block, i.e. i == kept[i] (skipped as an identity move). Processing ranks in ascending chunks
// of kChunk rows, with every read of a chunk completed (CTA barrier) before any write of it,
// is therefore hazard-free: writes of chunk j land on logical positions < (j+1)*kChunk, below
// every source of chunks > j. Rows move as 16-byte vectors, coalesced along d.
#include "internal.h"

namespace zpc {
namespace {

constexpr int kThreads = 256;
constexpr int kChunk = 64;           // rows per chunk
constexpr int kMaxVecPerRow = 32;    // d*e/16 <= 32 (fp32, d=128)
constexpr int kRegs = kChunk * kMaxVecPerRow / kThreads;   // 8 int4 per tensor per thread

__global__ void __launch_bounds__(kThreads) k_compact(Call c) {
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
  const size_t row_vecs = (size_t)vpr;
  unsigned moved = 0;

  for (int base = 0; base < ell; base += kChunk) {
    int4 kb[kRegs], vb[kRegs];
    size_t dst[kRegs];
    const int rows = min(kChunk, ell - base);
    const int nvec = rows * vpr;
#pragma unroll
    for (int k = 0; k < kRegs; ++k) {
      const int v = threadIdx.x + k * kThreads;
      dst[k] = (size_t)-1;
      if (v < nvec) {
        const int i = base + v / vpr, e = v % vpr;
        const int t = kept[i];
        const int sblk = table[t / c.b], dblk = tg[i / c.b];
        const size_t src = kv_row(c, l, sblk, t % c.b, h) * esz / 16 + e;
        const size_t d = kv_row(c, l, dblk, i % c.b, h) * esz / 16 + e;
        if (src != d) {
          kb[k] = K[src];
          vb[k] = V[src];
          dst[k] = d;
        }
      }
    }
    __syncthreads();   // all reads of this chunk precede any write of it
#pragma unroll
    for (int k = 0; k < kRegs; ++k) {
      if (dst[k] != (size_t)-1) {
        Kw[dst[k]] = kb[k];
        Vw[dst[k]] = vb[k];
        moved += ((threadIdx.x + k * kThreads) % vpr) == 0;
      }
    }
  }
  (void)row_vecs;
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
