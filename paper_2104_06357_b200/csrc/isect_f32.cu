// isect_f32.cu — float instantiations of the fused intersection kernel.
#include "isect_kernel.cuh"

namespace sd {
SD_ISECT_DISPATCH(float)
}  // namespace sd
