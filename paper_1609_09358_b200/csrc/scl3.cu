// scl3.cu -- K3 v3 host side: layout, eligibility, dispatch (kernel: scl3.cuh).
#include "args.cuh"
#include "scl3_decl.cuh"


namespace pc {

using s3::llo;
using s3::pso;
using s3::T;

bool scl3_eligible(const SclArgs &a, int L)
{
    (void)L;
    return a.code.n >= s3::T + 1 && a.code.n <= 12;
}

int scl3_prepare(SclArgs &a, int L, int nv_req)
{
    const int n = a.code.n;
    // stored LLR levels T+1..tp need 5-bit pointers in 32 bits (<= 6 levels)
    int nv = nv_req < 0 ? 0 : nv_req;
    const int nv_max = n - 2 - T > 0 ? n - 2 - T : 0; // keep level T+1 stored (or the channel)
    const int nv_min = n - 1 - (T + 6) > 0 ? n - 1 - (T + 6) : 0;
    if (nv > nv_max)
        nv = nv_max;
    if (nv < nv_min)
        nv = nv_min;
    if (nv > 4)
        return PC_ERR_UNSUPPORTED;
    a.nv = nv;
    a.tp = n - 1 - nv;
    const int lw = a.tp >= T + 1 ? llo(a.tp + 1) : 0;
    a.ss = ((lw + 7) & ~7) + 4; // stride = 4 (mod 8) floats: the 8 lanes of an LDS.128 phase hit distinct banks
    a.psw = pso(n) | 1;
    a.uhs = (a.code.k + 31) >> 5; // traceback windows W
    const int W = a.uhs;
    const int F = 32 / L;
    int o = 32 * a.ss;
    a.o_ps = o;
    o += 32 * a.psw;
    a.o_tb = a.o_tba = -1; // the traceback lives in the workspace (scl3_workspace_bytes)
    a.o_cand = o;
    o += 128; // per group 4L words: candidate metrics + indices
    a.o_wrow = o;
    o += (F * W + 3) & ~3;
    // Channel LLRs stay in global memory (L1/L2): staging them in shared memory
    // costs a warp per SM and measured slower (tools/scl_ab.py, round 1).
    const bool ch_smem = false;
    a.o_ch = ch_smem ? o : -1;
    if (ch_smem)
        o += F * a.code.N;
    a.warp_words = (o + 3) & ~3;
    a.table_words = 0;
    // The frozen prefix is decoded element-parallel in the slots of lanes 1..31
    // (unused while one path is alive): two ping-pong buffers of N floats.
    a.prefix = (L == 32 && 2 * a.code.N <= 31 * a.ss && a.code.first_info > 0) ? 1 : 0;
    return PC_OK;
}

// Upper bound of the resident warps of a K3 v3 launch (shared memory is its
// occupancy limit) times the per-warp traceback, plus the counter block.
int64_t scl3_workspace_bytes(const SclArgs &a, int L, int wpc)
{
    (void)L;
    if (wpc < 1 || wpc > 4)
        wpc = 1;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    const int64_t per_cta = (int64_t)wpc * a.warp_words * 4 + 1024; // + the per-CTA reservation
    int64_t ctas = (228 * 1024) / per_cta;
    if (ctas > 32)
        ctas = 32;
    int64_t warps = ctas * wpc;
    if (warps > 64)
        warps = 64;
    if (warps < wpc)
        warps = wpc;
    return 256 + (int64_t)sms * warps * a.uhs * 40 * 4;
}

int launch_scl3(const SclArgs &a, int L, int wpc, cudaStream_t s)
{
    if (a.B == 0)
        return PC_OK;
    if (cudaMemsetAsync(a.work, 0, sizeof(int32_t), s) != cudaSuccess)
        return PC_ERR_CUDA;
    const int F = 32 / L;
    const int max_warps = (a.B + F - 1) / F;
    if (wpc < 1 || wpc > 4)
        wpc = 1;
    switch (L) {
    case 1: return launch_scl3_for<1>(a, wpc, max_warps, s);
    case 2: return launch_scl3_for<2>(a, wpc, max_warps, s);
    case 4: return launch_scl3_for<4>(a, wpc, max_warps, s);
    case 8: return launch_scl3_for<8>(a, wpc, max_warps, s);
    case 16: return launch_scl3_for<16>(a, wpc, max_warps, s);
    case 32: return launch_scl3_for<32>(a, wpc, max_warps, s);
    default: return PC_ERR_UNSUPPORTED;
    }
}

} // namespace pc
