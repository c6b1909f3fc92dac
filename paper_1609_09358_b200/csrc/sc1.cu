// sc1.cu -- K3 for list size 1 (successive cancellation, reference sim.py:152-153:
// SC is scl_decode with L = 1): one WARP per frame (sm_100a).
//
// K3 v3 (scl3.cuh) maps 32 / L frames onto a warp, one lane per path, so at
// L = 1 every lane walks a whole frame alone: the upper tree levels (2^s
// elements each) run serially per lane, 32 channel rows stream through L1/L2
// per warp, and one frame takes ~0.8 ms at N = 2048.  Here the 32 lanes of a
// warp share one frame:
//   * the channel row is staged in the warp's shared memory;
//   * every upper level (5 .. n-1) is computed element-parallel by the warp
//     (lane t: elements t, t + 32, ...), f or g with the stored partial sums;
//   * each block of 32 leaves runs on lane 0 from registers with the same leaf
//     code as K3 v3 (levels 4..0, their partial sums in one word, the fp32
//     metric and the L = 1 decision rule c1 < c0 of the (metric, index) order,
//     _kernels.py:247-311), so decisions, metric and CRC flag are bit-identical
//     to K3 v3 at L = 1 (tests/test_gpu_scl.py);
//   * the block's codeword is folded into the stored partial sums
//     element-parallel.
// Shared memory per warp: channel N floats, levels 5..n-1 (N - 32 floats),
// partial sums N/32 words, decisions N/32 words.
#include "args.cuh"
#include "scl_math.cuh"

namespace pc {

namespace sc1 {
constexpr int T = 5; // leaf blocks of 32
__host__ __device__ constexpr int lvl(int s) { return (1 << s) - 32; }      // level s >= 5, floats
__host__ __device__ constexpr int pso(int s) { return (1 << (s - 5)) - 1; } // partial sums of level s >= 5, words
__host__ __device__ inline int warp_floats(int N) { return 2 * N + 2 * (N / 32) + 4; }
} // namespace sc1

template <bool FEX>
__global__ void __launch_bounds__(128) k_sc1(const SclArgs a)
{
    using namespace sc1;
    constexpr uint32_t FULL = 0xffffffffu;
    extern __shared__ __align__(16) float smf[];
    const int N = a.code.N, n = a.code.n;
    const int lane = threadIdx.x & 31;
    float *ch = smf + (size_t)(threadIdx.x >> 5) * warp_floats(N);
    float *lv = ch + N;
    uint32_t *ps = reinterpret_cast<uint32_t *>(lv + N);
    uint32_t *ub = ps + N / 32;
    const uint32_t *frzg = a.code.frozen_bits;
    const uint32_t *damg = a.code.da_bits;
    const uint32_t *colg = a.code.crc_cols;
    const bool use_crc = a.code.crc_width > 0;
    const int total = a.count != nullptr ? *a.count : a.B;
    const int nblk = N >> T;

    for (;;) {
        int qi = 0;
        if (lane == 0)
            qi = atomicAdd(a.work, 1);
        qi = __shfl_sync(FULL, qi, 0);
        if (qi >= total)
            break;
        const int frame = a.queue != nullptr ? a.queue[qi] : qi;
        {
            const float4 *g = reinterpret_cast<const float4 *>(a.llr + (size_t)frame * N);
            for (int t = lane; t < N / 4; t += 32)
                reinterpret_cast<float4 *>(ch)[t] = __ldg(g + t);
        }
        __syncwarp();
        float metric = 0.0f;
        uint32_t syn = 0u;
        for (int b = 0; b < nblk; ++b) {
            const int i0 = b << T;
            // ---- upper descent: levels start..5, element-parallel ----
            const int start = (b == 0) ? n - 1 : T + __ffs(b) - 1;
            for (int s = start; s >= T; --s) {
                const int w = 1 << s;
                const float *src = (s + 1 == n) ? ch : lv + lvl(s + 1);
                float *dst = lv + lvl(s);
                if ((i0 >> s) & 1) {
                    const uint32_t *pw = ps + pso(s);
                    for (int t = lane; t < w; t += 32)
                        dst[t] = scl_g(src[t], src[t + w], (pw[t >> 5] >> (t & 31)) & 1u);
                } else {
                    for (int t = lane; t < w; t += 32)
                        dst[t] = scl_f<FEX>(src[t], src[t + w]);
                }
                __syncwarp();
            }
            // ---- the block's 32 leaves on lane 0, registers only (K3 v3's leaf code at L = 1) ----
            uint32_t betaT = 0;
            if (lane == 0) {
                float x[32];
#pragma unroll
                for (int t = 0; t < 32; t += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(lv + t);
                    x[t] = v.x, x[t + 1] = v.y, x[t + 2] = v.z, x[t + 3] = v.w;
                }
                const uint32_t fzw = __ldg(frzg + b);
                const uint32_t daw = damg != nullptr ? __ldg(damg + b) : 0u;
                float l4[16], l3[8], l2[4], l1[2];
                uint32_t psr = 0, bu = 0;
#pragma unroll 1
                for (int j = 0; j < 32; ++j) {
                    float lam;
                    if (j & 1) {
                        lam = scl_g(l1[0], l1[1], psr & 1u);
                    } else {
                        if (j & 2) {
                            l1[0] = scl_g(l2[0], l2[2], (psr >> 1) & 1u);
                            l1[1] = scl_g(l2[1], l2[3], (psr >> 2) & 1u);
                        } else {
                            if (j & 4) {
#pragma unroll
                                for (int t = 0; t < 4; ++t)
                                    l2[t] = scl_g(l3[t], l3[t + 4], (psr >> (3 + t)) & 1u);
                            } else {
                                if (j & 8) {
#pragma unroll
                                    for (int t = 0; t < 8; ++t)
                                        l3[t] = scl_g(l4[t], l4[t + 8], (psr >> (7 + t)) & 1u);
                                } else {
                                    if (j & 16) {
#pragma unroll
                                        for (int t = 0; t < 16; ++t)
                                            l4[t] = scl_g(x[t], x[t + 16], (psr >> (15 + t)) & 1u);
                                    } else {
#pragma unroll
                                        for (int t = 0; t < 16; ++t)
                                            l4[t] = scl_f<FEX>(x[t], x[t + 16]);
                                    }
#pragma unroll
                                    for (int t = 0; t < 8; ++t)
                                        l3[t] = scl_f<FEX>(l4[t], l4[t + 8]);
                                }
#pragma unroll
                                for (int t = 0; t < 4; ++t)
                                    l2[t] = scl_f<FEX>(l3[t], l3[t + 4]);
                            }
                            l1[0] = scl_f<FEX>(l2[0], l2[2]);
                            l1[1] = scl_f<FEX>(l2[1], l2[3]);
                        }
                        lam = scl_f<FEX>(l1[0], l1[1]);
                    }
                    const uint32_t fz = (fzw >> j) & 1u, dz = (daw >> j) & 1u;
                    float inc0, inc1;
                    metric_incs(lam, a.metric_exact, inc0, inc1);
                    uint32_t u;
                    if (fz | dz) {
                        u = (dz && lam < 0.0f) ? 1u : 0u;
                        metric += u ? inc1 : inc0;
                    } else {
                        // one path: keep the better child, a tie keeps u = 0 (candidate
                        // index 0 < 1, _kernels.py:253-267)
                        const float c0 = metric + inc0, c1 = metric + inc1;
                        u = c1 < c0 ? 1u : 0u;
                        metric = u ? c1 : c0;
                    }
                    if (!fz && u && use_crc)
                        syn ^= __ldg(colg + i0 + j);
                    bu |= u << j;
                    // fold u into the register partial sums: level S = trailing ones of j
                    uint32_t Fw = u;
                    if (j & 1) {
                        Fw = ((psr ^ Fw) & 1u) | (Fw << 1);
                        if (j & 2) {
                            Fw = (((psr >> 1) ^ Fw) & 3u) | (Fw << 2);
                            if (j & 4) {
                                Fw = (((psr >> 3) ^ Fw) & 15u) | (Fw << 4);
                                if (j & 8) {
                                    Fw = (((psr >> 7) ^ Fw) & 255u) | (Fw << 8);
                                    if (j & 16)
                                        betaT = (((psr >> 15) ^ Fw) & 0xffffu) | (Fw << 16);
                                    else
                                        psr = (psr & ~(0xffffu << 15)) | (Fw << 15);
                                } else {
                                    psr = (psr & ~(255u << 7)) | (Fw << 7);
                                }
                            } else {
                                psr = (psr & ~(15u << 3)) | (Fw << 3);
                            }
                        } else {
                            psr = (psr & ~(3u << 1)) | (Fw << 1);
                        }
                    } else {
                        psr = (psr & ~1u) | Fw;
                    }
                }
                ub[b] = bu;
            }
            // ---- block end: fold the block codeword into the stored partial sums ----
            betaT = __shfl_sync(FULL, betaT, 0);
            const int S = T + __ffs(~b) - 1; // level of the node this block completes
            if (S < n) {
                const int words = 1 << (S - T);
                for (int w = lane; w < words; w += 32) {
                    uint32_t v = betaT;
                    for (int s = T; s < S; ++s)
                        if (((w >> (s - T)) & 1) == 0)
                            v ^= ps[pso(s) + (w & ((1 << (s - T)) - 1))];
                    ps[pso(S) + w] = v;
                }
            }
            __syncwarp();
        }
        // ---- outputs (the one path is the winner, scl.py:177-191) ----
        metric = __shfl_sync(FULL, metric, 0);
        syn = __shfl_sync(FULL, syn, 0);
        const int NW = N >> 5;
        if (a.u_bits != nullptr)
            for (int w = lane; w < NW; w += 32)
                a.u_bits[(size_t)frame * NW + w] = ub[w];
        if (a.payload != nullptr) {
            const int m = a.code.m, MW = (m + 31) >> 5;
            for (int bb = lane; bb < 32 * MW; bb += 32) {
                uint32_t bit = 0u;
                if (bb < m) {
                    const int p = __ldg(a.code.info_pos + bb);
                    bit = (ub[p >> 5] >> (p & 31)) & 1u;
                }
                const uint32_t v = __ballot_sync(FULL, bit);
                if (lane == 0)
                    a.payload[(size_t)frame * MW + (bb >> 5)] = v;
            }
        }
        if (lane == 0) {
            const bool ok = use_crc && syn == a.code.crc_offset;
            if (a.metric != nullptr)
                a.metric[frame] = metric;
            if (a.crc_ok != nullptr)
                a.crc_ok[frame] = ok;
            if (a.sel != nullptr)
                a.sel[frame] = ok;
            if (a.t_done != nullptr)
                a.t_done[frame] = globaltimer();
        }
        __syncwarp();
    }
}

bool sc1_eligible(const SclArgs &a) { return a.code.n >= 6 && a.code.n <= 12; }

int launch_sc1(const SclArgs &a, cudaStream_t s)
{
    if (a.B == 0)
        return PC_OK;
    if (cudaMemsetAsync(a.work, 0, sizeof(int32_t), s) != cudaSuccess)
        return PC_ERR_CUDA;
    auto kern = a.f_exact ? k_sc1<true> : k_sc1<false>;
    const int N = a.code.N;
    const size_t per_warp = (size_t)sc1::warp_floats(N) * 4;
    int wpc = 4;
    while (wpc > 1 && (size_t)wpc * per_warp > 200 * 1024)
        --wpc;
    const size_t smem = (size_t)wpc * per_warp;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return PC_ERR_CUDA;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpc, smem) != cudaSuccess || per_sm < 1)
        return PC_ERR_UNSUPPORTED;
    long long grid = (long long)sms * per_sm;
    const long long need = ((long long)a.B + wpc - 1) / wpc; // one warp per frame at most
    if (grid > need)
        grid = need;
    kern<<<(int)grid, 32 * wpc, smem, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

} // namespace pc
