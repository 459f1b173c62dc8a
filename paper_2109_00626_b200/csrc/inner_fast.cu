// inner_fast.cu -- specialised tt_inner kernels (filled in after the generic path is parity-green).
#include "ttc_internal.h"

namespace ttc {

bool inner_fast_supported(const InnerArgs&, int, bool) { return false; }

cudaError_t launch_inner_fast(const InnerArgs&, int, bool, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace ttc
