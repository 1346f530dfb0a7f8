// placeholder, replaced by the tcgen05 int8-limb leaf kernel
#include "wm_device.h"
namespace wm {
bool leaf_i8_supported(const MulParams&) { return false; }
cudaError_t launch_leaf_i8(const MulParams&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace wm
