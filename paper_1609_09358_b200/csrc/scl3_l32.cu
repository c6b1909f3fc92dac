// scl3_l32.cu -- K3 v3 kernels for list size 32 (see scl3.cuh).
#include "scl3.cuh"

namespace pc {
template int launch_scl3_for<32>(const SclArgs &a, int wpc, int max_warps, cudaStream_t s);
} // namespace pc

#ifdef SCL3_STATS
// development aid (tools/scl3_stats.py): read and clear the L = 32 kernels' counters
extern "C" int pc_debug_scl3_stats(unsigned long long *out)
{
    if (cudaMemcpyFromSymbol(out, pc::g_scl3_stats, sizeof(unsigned long long) * 8) != cudaSuccess)
        return -1;
    unsigned long long z[8] = {};
    return cudaMemcpyToSymbol(pc::g_scl3_stats, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif
