// K2 (INT4) -- placeholder until the kind::i8 kernel lands.
#include "k1_launch.h"

namespace svdq {
cudaError_t launch_k2_int4(const K2Maps &, const K2Params &, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace svdq
