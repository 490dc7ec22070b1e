// k_batch.cu -- K5: many independent HALP problems, one persistent CTA each.
#include "halp_device.cuh"
#include "kernels.h"

namespace halp {
cudaError_t launch_batch(const BatchParams&, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace halp
