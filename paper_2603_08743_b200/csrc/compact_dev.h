// Device code of a5 (in-place compaction of one unit's kept K/V rows, Alg. 4), shared by
// k_compact (compact.cu). See compact.cu for the hazard argument.
#pragma once
#include "internal.h"

namespace zpc {
namespace {

template <int VPR, int kVec>
struct Chunk {
  int4 k[kVec], v[kVec];
  uint32_t dst[kVec];                // destination vector index within the layer-head plane, ~0u = none
  float f[kVec];                     // NEXT-2: the row's global score (the row's first vector carries it)
  uint32_t fdst[kVec];               // its destination row (blk*b + slot), ~0u = none
};

template <int VPR, int kVec, int kThreads>
__device__ __forceinline__ void load_chunk(const Call& c, Chunk<VPR, kVec>& ch, int base, int ell, const int32_t* kept,
                                           const int32_t* table, const int32_t* tg, const int4* K, const int4* V,
                                           size_t plane, int bsh, const float* F, size_t fplane) {
  constexpr int CH = kVec * kThreads / VPR;        // ranks per chunk
  const int nvec = min(CH, ell - base) * VPR;
  const uint32_t rowv = (uint32_t)c.h_kv * VPR;    // vectors between consecutive slots
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    const int v = threadIdx.x + k * kThreads;
    ch.dst[k] = ~0u;
    if (v < nvec) {
      const int i = base + v / VPR, e = v % VPR;
      const int t = kept[i];
      int sblk, sslot, dblk, dslot;
      if (bsh >= 0) {
        sblk = table[t >> bsh]; sslot = t & ((1 << bsh) - 1);
        dblk = tg[i >> bsh];    dslot = i & ((1 << bsh) - 1);
      } else {
        sblk = table[t / c.b]; sslot = t % c.b;
        dblk = tg[i / c.b];    dslot = i % c.b;
      }
      ZPC_CHECK(t >= i && sblk >= 0 && sblk < c.N_total && dblk >= 0 && dblk < c.N_total);
      // vector index relative to the (layer, head) plane: (blk*b + slot)*h_kv*VPR + e
      const uint32_t src = ((uint32_t)sblk * c.b + sslot) * rowv + e;
      const uint32_t d = ((uint32_t)dblk * c.b + dslot) * rowv + e;
      ch.fdst[k] = ~0u;
      if (src != d) {
        ch.k[k] = K[plane + src];
        ch.v[k] = V[plane + src];
        ch.dst[k] = d;
        if (F && e == 0) {            // F moves with its K/V row
          ch.f[k] = F[fplane + ((size_t)sblk * c.b + sslot) * c.h_kv];
          ch.fdst[k] = (uint32_t)dblk * c.b + dslot;
        }
      }
    }
  }
}

// the addresses of one chunk: kept[i] -> table -> source slot, targets -> destination slot (a chain of
// dependent L2 reads), computed one chunk ahead of the K/V loads that use them
template <int kVec>
struct ChunkIdx {
  uint32_t src[kVec], dst[kVec];     // vector indices within the layer-head plane; dst ~0u = none
  uint32_t fsrc[kVec], fdst[kVec];   // NEXT-2: F row indices (blk*b + slot); fdst ~0u = none
};
template <int VPR, int kVec, int kThreads, bool HasF>
__device__ __forceinline__ void load_idx(const Call& c, ChunkIdx<kVec>& ix, int base, int ell, const int32_t* kept,
                                         const int32_t* table, const int32_t* tg, int bsh) {
  constexpr int CH = kVec * kThreads / VPR;        // ranks per chunk
  const int nvec = min(CH, ell - base) * VPR;
  const uint32_t rowv = (uint32_t)c.h_kv * VPR;    // vectors between consecutive slots
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    const int v = threadIdx.x + k * kThreads;
    ix.dst[k] = ~0u;
    if (HasF) ix.fdst[k] = ~0u;
    if (v < nvec) {
      const int i = base + v / VPR, e = v % VPR;
      const int t = kept[i];
      int sblk, sslot, dblk, dslot;
      if (bsh >= 0) {
        sblk = table[t >> bsh]; sslot = t & ((1 << bsh) - 1);
        dblk = tg[i >> bsh];    dslot = i & ((1 << bsh) - 1);
      } else {
        sblk = table[t / c.b]; sslot = t % c.b;
        dblk = tg[i / c.b];    dslot = i % c.b;
      }
      ZPC_CHECK(t >= i && sblk >= 0 && sblk < c.N_total && dblk >= 0 && dblk < c.N_total);
      const uint32_t src = ((uint32_t)sblk * c.b + sslot) * rowv + e;
      const uint32_t d = ((uint32_t)dblk * c.b + dslot) * rowv + e;
      if (src != d) {
        ix.src[k] = src;
        ix.dst[k] = d;
        if (HasF && e == 0) {         // F moves with its K/V row
          ix.fsrc[k] = (uint32_t)sblk * c.b + sslot;
          ix.fdst[k] = (uint32_t)dblk * c.b + dslot;
        }
      }
    }
  }
}
template <int VPR, int kVec, bool HasF>
__device__ __forceinline__ void load_data(Chunk<VPR, kVec>& ch, const ChunkIdx<kVec>& ix, const int4* K, const int4* V,
                                          size_t plane, const float* F, size_t fplane, int h_kv) {
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    ch.dst[k] = ix.dst[k];
    if (HasF) ch.fdst[k] = ix.fdst[k];
    if (ix.dst[k] != ~0u) {
      ch.k[k] = K[plane + ix.src[k]];
      ch.v[k] = V[plane + ix.src[k]];
      if (HasF && ix.fdst[k] != ~0u) ch.f[k] = F[fplane + (size_t)ix.fsrc[k] * h_kv];
    }
  }
}

// the compaction of unit `unit` by the kThreads threads of the calling CTA (kept list and new_lens in place)
// Ahead: the index chain of chunk j + 2 runs a chunk ahead of the K/V loads (launch_compact picks it per call)
template <int VPR, int kVec, int kThreads, bool HasF, bool Ahead>
__device__ __forceinline__ void compact_unit(const Call& c, const int unit) {
  constexpr int CH = kVec * kThreads / VPR;
  const int h = unit % c.h_kv;
  const int l = (unit / c.h_kv) % c.L;
  const int r = unit / (c.h_kv * c.L);
  const int ell = c.new_lens[unit];
  const int nm1 = c.n_max - 1;
  const int32_t* kept = c.ws.kept + (size_t)unit * c.ws.kept_stride;
  const int32_t* tg = c.ws.targets + (size_t)r * nm1;
  const int32_t* table = c.tables + (size_t)r * c.table_stride;
  const int bsh = (c.b & (c.b - 1)) == 0 ? __ffs(c.b) - 1 : -1;
  const int4* K = reinterpret_cast<const int4*>(c.k_cache);
  const int4* V = reinterpret_cast<const int4*>(c.v_cache);
  int4* Kw = reinterpret_cast<int4*>(c.k_cache);
  int4* Vw = reinterpret_cast<int4*>(c.v_cache);
  // start of the (layer l, head h) plane in vectors; per-row offsets are 32-bit within a layer
  const size_t plane = (size_t)l * c.N_total * c.b * c.h_kv * VPR + (size_t)h * VPR;
  float* Fw = HasF ? c.f_cache : nullptr;   // NEXT-2 relocation (HasF: ZPC_F_GLOBAL_SCORE)
  const size_t fplane = (size_t)l * c.N_total * c.b * c.h_kv + h;
  unsigned moved = 0;

  if constexpr (Ahead) {
    // three stages per iteration: stores of chunk j, K/V loads of chunk j + 1 (addresses ready), index chain of
    // chunk j + 2. Chunk j + 1's sources are at positions >= (j + 1) * CH, above every write of chunk j (the hazard
    // argument of compact.cu), so its loads may be in flight while chunk j is stored; the index reads touch
    // kept / tables / targets only, which the compaction never writes.
    Chunk<VPR, kVec> cur, nxt;
    ChunkIdx<kVec> ix;                 // the addresses of chunk j + 1 (consumed by its loads, then chunk j + 2's)
    if (ell > 0) {
      load_idx<VPR, kVec, kThreads, HasF>(c, ix, 0, ell, kept, table, tg, bsh);
      load_data<VPR, kVec, HasF>(cur, ix, K, V, plane, Fw, fplane, c.h_kv);
      if (CH < ell) load_idx<VPR, kVec, kThreads, HasF>(c, ix, CH, ell, kept, table, tg, bsh);
    }
    for (int base = 0; base < ell; base += CH) {
      __syncthreads();   // every read of chunk `base` has returned before any write of it
      const bool more = base + CH < ell;
      if (more) load_data<VPR, kVec, HasF>(nxt, ix, K, V, plane, Fw, fplane, c.h_kv);
#pragma unroll
      for (int k = 0; k < kVec; ++k) {
        if (cur.dst[k] != ~0u) {
          Kw[plane + cur.dst[k]] = cur.k[k];
          Vw[plane + cur.dst[k]] = cur.v[k];
          if (HasF && cur.fdst[k] != ~0u) Fw[fplane + (size_t)cur.fdst[k] * c.h_kv] = cur.f[k];
          moved += ((threadIdx.x + k * kThreads) % VPR) == 0;
        }
      }
      if (base + 2 * CH < ell) load_idx<VPR, kVec, kThreads, HasF>(c, ix, base + 2 * CH, ell, kept, table, tg, bsh);
      if (more) cur = nxt;
    }
  } else {
    Chunk<VPR, kVec> cur, nxt;
    if (ell > 0) load_chunk<VPR, kVec, kThreads>(c, cur, 0, ell, kept, table, tg, K, V, plane, bsh, Fw, fplane);
    for (int base = 0; base < ell; base += CH) {
      __syncthreads();   // every read of chunk `base` has returned before any write of it
      const bool more = base + CH < ell;
      if (more) load_chunk<VPR, kVec, kThreads>(c, nxt, base + CH, ell, kept, table, tg, K, V, plane, bsh, Fw, fplane);
#pragma unroll
      for (int k = 0; k < kVec; ++k) {
        if (cur.dst[k] != ~0u) {
          Kw[plane + cur.dst[k]] = cur.k[k];
          Vw[plane + cur.dst[k]] = cur.v[k];
          if (cur.fdst[k] != ~0u) Fw[fplane + (size_t)cur.fdst[k] * c.h_kv] = cur.f[k];
          moved += ((threadIdx.x + k * kThreads) % VPR) == 0;
        }
      }
      if (more) cur = nxt;
    }
  }
  if (c.flags & ZPC_F_COUNT_MOVES) {
    for (int o = 16; o; o >>= 1) moved += __shfl_xor_sync(0xffffffffu, moved, o);
    if ((threadIdx.x & 31) == 0 && moved) atomicAdd(c.ws.moves, (unsigned long long)moved);
  }
}

}  // namespace
}  // namespace zpc
