// a5: in-place compaction of kept K/V rows (Alg. 4), one CTA per unit (r, l, h).
//
// Alg. 4 is a sequential two-pointer sweep; here rank i of the ascending kept list moves
// row kept[i] -> target slot i. Hazard argument: kept[i] >= i, and a destination
// aliases a source only when both are the same logical position of an own target block, i.e.
// i == kept[i] (skipped as an identity move). Ranks are processed in ascending chunks with every
// read of a chunk completed (CTA barrier) before any write of it; the writes of chunk j land on
// logical positions < (j+1)*chunk, below every source of chunks > j, so the loads of chunk j+1
// are issued before the stores of chunk j (software pipelining).
// Rows move as 16-byte vectors, coalesced along d; a chunk is kVec vectors per tensor per thread
// (VPR = vectors per row is a template parameter). HBM-bound: the bytes in flight per SM decide
// the rate: one vector per thread, CTA width chosen per call so ~2048 threads per SM are in flight
// (launch_compact).
#include <cstdlib>

#include "compact_dev.h"
#include "internal.h"

namespace zpc {
namespace {


template <int VPR, int kVec, int kThreads, int kMinCtas, bool HasF, bool Ahead>
__global__ void __launch_bounds__(kThreads, kMinCtas) k_compact(Call c) {
  if (*c.status != ZPC_OK) return;
  compact_unit<VPR, kVec, kThreads, HasF, Ahead>(c, blockIdx.x);
}

}  // namespace

cudaError_t launch_compact(const Call& c, cudaStream_t s) {
  const int units = c.R * c.L * c.h_kv;
  if (units == 0) return cudaSuccess;
  const int vpr = c.d * (c.dtype == ZPC_BF16 ? 2 : 4) / 16;   // head_dim is 64 or 128 (validated)
  // One CTA per unit; the CTA width is picked so the threads in flight per SM stay near 2048 (the copy
  // is latency-bound: bytes in flight per SM decide the rate, and deeper per-thread buffering measured
  // slower than more threads: 7B shape 1 vector/thread at 16 CTAs/SM 2.60 ms, 2 @ 8: 2.88, 4 @ 5: 3.21).
  // A/B on one B200 (ZPC_COMPACT_NT, compact ms by CTA width 128 / 256 / 512 / 1024):
  //   paper_op 1 request  (288 units,  ~2 per SM): 0.336 / 0.201 / 0.143 / 0.117
  //   paper_op 2 requests (576 units,  ~4 per SM): 0.373 / 0.266 / 0.219 / 0.230
  //   paper_op 4 requests (1152 units, ~8 per SM): 0.495 / 0.402 / 0.429 / 0.453
  //   qwen7b 64 requests  (7168 units, 48 per SM): 2.620 / 2.535 / 2.672 / 2.772
  int dev = 0, sms = 0;   // queried per call (the current device's SM count; no cached state)
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return cudaErrorInvalidDevice;
  int nt = units >= sms * 6 ? 256 : (units >= sms * 3 ? 512 : 1024);
  const uint32_t vnt = (c.variant >> ZPC_V_COMPACT_SHIFT) & 7u;   // params.variant override (tests, A/B)
  if (vnt != 0) nt = 64 << vnt;
  const bool hf = (c.flags & ZPC_F_GLOBAL_SCORE) != 0;   // NEXT-2: F rows move with K/V
  // the index chain a chunk ahead (compact_dev.h) except for 256-wide CTAs over large blocks. A/B on one B200,
  // compact ms old / index-ahead by CTA width 128 / 256 / 512 / 1024:
  //   qwen7b (b = 16, 7168 units):        2.63 / 2.60, 2.54 / 2.48, 2.64 / 2.46, -
  //   paper_op 4 requests (b = 256):      0.480 / 0.483, 0.396 / 0.437, 0.417 / 0.406, 0.437 / 0.413
  //   paper_op 1 request (b = 256):       -, 0.193 / 0.178, 0.140 / 0.135, 0.114 / 0.111
  const bool ahead = !(c.b >= 128 && nt == 256);
  // __launch_bounds__ keeps 2048 threads per SM (32 registers; 12-84 B of spills, L1-resident). 1536 threads per
  // SM without most spills (40 registers) measured slower: qwen7b 2.48 -> 2.54 ms, paper_op 0.395 -> 0.499,
  // llama8b 1.48 -> 1.50
#define ZPC_COMPACT_NT(VPR, HF)                                                                   \
  if (nt == 128) k_compact<VPR, 1, 128, 16, HF, true><<<units, 128, 0, s>>>(c);                  \
  else if (nt == 256 && ahead) k_compact<VPR, 1, 256, 8, HF, true><<<units, 256, 0, s>>>(c);     \
  else if (nt == 256) k_compact<VPR, 1, 256, 8, HF, false><<<units, 256, 0, s>>>(c);             \
  else if (nt == 512) k_compact<VPR, 1, 512, 4, HF, true><<<units, 512, 0, s>>>(c);              \
  else k_compact<VPR, 1, 1024, 2, HF, true><<<units, 1024, 0, s>>>(c);
#define ZPC_COMPACT_CASE(VPR)                                                             \
  case VPR:                                                                              \
    if (hf) { ZPC_COMPACT_NT(VPR, true) } else { ZPC_COMPACT_NT(VPR, false) }            \
    break;
  switch (vpr) {
    ZPC_COMPACT_CASE(8)
    ZPC_COMPACT_CASE(16)
    ZPC_COMPACT_CASE(32)
    default: return cudaErrorInvalidValue;
  }
#undef ZPC_COMPACT_CASE
#undef ZPC_COMPACT_NT
  return cudaGetLastError();
}

}  // namespace zpc
