// isect_f64.cu — double instantiations of the fused intersection kernel.
#include "isect_kernel.cuh"

namespace sd {
SD_ISECT_DISPATCH(double)
}  // namespace sd
