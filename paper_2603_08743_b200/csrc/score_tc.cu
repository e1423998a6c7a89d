// a1 + a2 on tcgen05 tensor cores (bf16 pools): placeholder until the sm_100a kernel lands.
#include "internal.h"
namespace zpc {
cudaError_t launch_score_tc(const Call& c, cudaStream_t s, bool* used) {
  (void)c; (void)s;
  *used = false;
  return cudaSuccess;
}
}  // namespace zpc
