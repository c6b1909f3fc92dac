// scl3_l4.cu -- K3 v3 kernels for list size 4 (see scl3.cuh).
#include "scl3.cuh"

namespace pc {
template int launch_scl3_for<4>(const SclArgs &a, int wpc, int max_warps, cudaStream_t s);
} // namespace pc
