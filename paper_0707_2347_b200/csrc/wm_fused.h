// Fused schedule-run kernels (generated bodies in wm_fused_gen.cuh).
#pragma once

#include <cuda_runtime.h>

#include "wm_fused_gen.cuh"

namespace wm {
cudaError_t launch_group(int gid, const fused::GroupParams& G, bool real, cudaStream_t s,
                         unsigned long long* tl = nullptr);
}  // namespace wm
