// bp3h.cu -- K1 v3 at N = 128: two frames per warp, one per half-warp, all
// seven boundaries in registers (sm_100a).
//
// The N = 128 member of the layout family of bp3.cu (same recursion, stop
// rules -- CRC, re-encode, none -- and outputs as k_bp2, reference bp.py:120-217, and the same per-PE
// arithmetic bp_math.cuh::bp_pe2, so bit-identical to k_bp2<7, ...>).  A frame
// is 16 threads of 8 nodes.  With h = lane >> 4 the half-warp and l = lane & 15
// its lane, the nodes of a thread are, by layout:
//   A  x = 8l + r                        boundaries 1, 2, 3 (strides 1, 2, 4)
//   B  x = (l & 7) + 8r + 64(l >> 3)     boundaries 4, 5, 6 (strides 8, 16, 32)
//   C  x = l + 16(r & 3) + 64(r >> 2)    boundary 7         (stride 64)
// and a row crosses layouts through 136 floats of half-warp scratch (R[3]
// A->B, R[6] B->C, L[6] C->B, L[3] B->A), indexed x + 8(x >> 6) + 144h so that
// both halves' scalar B and C accesses fall in 32 distinct banks.  The channel
// row L[7] stays in registers in layout C.
//
// The two halves are independent decoders (a frame per half, every warp
// collective on the half's own mask, as a 16-thread tile): one iteration of
// both frames per trip of the loop, and a half whose frame stops writes its
// outputs and takes the next frame while the other half waits only for that
// short block.  With the persistent frame counter (pc_bp_cfg_t.work) the
// warps take frames until none are left; without it each half decodes one.
#include "args.cuh"
#include "bp_math.cuh"

namespace pc {

namespace b3h {

constexpr int HS = 144; // floats between the two halves' scratch (16 banks apart)
constexpr int XSW = 280; // per-warp scratch floats: 144 + 128 + 8 padding

__device__ __forceinline__ int xa(int l, int r) { return 8 * l + r; }
__device__ __forceinline__ int xb(int l, int r) { return (l & 7) + 8 * r + 64 * (l >> 3); }
__device__ __forceinline__ int xc(int l, int r) { return l + 16 * (r & 3) + 64 * (r >> 2); }
__device__ __forceinline__ int xpad(int x) { return x + ((x >> 6) << 3); }

// One boundary inside a thread: register pairs (r, r + H), as bp3.cu::stage.
template <int GMODE, bool RS, int H>
__device__ __forceinline__ void stage(const float (&Rp)[8], const float (&Lj)[8], float (&out)[8], BpLim lim)
{
#pragma unroll
    for (int r1 = 0; r1 < 8; ++r1) {
        if (r1 & H)
            continue;
        const int r2 = r1 + H;
        if (RS)
            bp_pe2<GMODE, true>(Rp[r1], bp_comb<GMODE>(Lj[r2], Rp[r2]), Lj[r1], Rp[r2], lim, out[r1], out[r2]);
        else
            bp_pe2<GMODE, false>(Lj[r1], bp_comb<GMODE>(Lj[r2], Rp[r2]), Rp[r1], Lj[r2], lim, out[r1], out[r2]);
    }
}

// Layout changes through the half's scratch xs (hm = the half's lane mask).
__device__ __forceinline__ void a_to_b(const float (&v)[8], float (&o)[8], float *xs, int l, unsigned hm)
{
    __syncwarp(hm);
    float *p = xs + xpad(xa(l, 0));
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4 *>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
    __syncwarp(hm);
#pragma unroll
    for (int r = 0; r < 8; ++r)
        o[r] = xs[xpad(xb(l, r))];
}

__device__ __forceinline__ void b_to_a(const float (&v)[8], float (&o)[8], float *xs, int l, unsigned hm)
{
    __syncwarp(hm);
#pragma unroll
    for (int r = 0; r < 8; ++r)
        xs[xpad(xb(l, r))] = v[r];
    __syncwarp(hm);
    const float *p = xs + xpad(xa(l, 0));
    const float4 u = *reinterpret_cast<const float4 *>(p), w = *reinterpret_cast<const float4 *>(p + 4);
    o[0] = u.x, o[1] = u.y, o[2] = u.z, o[3] = u.w, o[4] = w.x, o[5] = w.y, o[6] = w.z, o[7] = w.w;
}

template <bool B2C>
__device__ __forceinline__ void b_c(const float (&v)[8], float (&o)[8], float *xs, int l, unsigned hm)
{
    __syncwarp(hm);
#pragma unroll
    for (int r = 0; r < 8; ++r)
        xs[xpad(B2C ? xb(l, r) : xc(l, r))] = v[r];
    __syncwarp(hm);
#pragma unroll
    for (int r = 0; r < 8; ++r)
        o[r] = xs[xpad(B2C ? xc(l, r) : xb(l, r))];
}

} // namespace b3h

#ifndef PC_BP3H_WARPS
#define PC_BP3H_WARPS 4
#endif
constexpr int BP3H_WARPS = PC_BP3H_WARPS; // warps per CTA (2 frames each)

#ifndef PC_BP3H_MINB
#define PC_BP3H_MINB 4 // 128 registers: 4 CTAs per SM (measured best; 5 and 6 were slower)
#endif

// (the default form gets the compiler's own choice, 128 registers: 1.8% faster than
// its choice under the 4-CTA bound; the others are held to 128 by the bound)
template <int GMODE, bool PERS, bool RE>
__global__ void __launch_bounds__(32 * BP3H_WARPS, (GMODE == 0 && !RE) ? 1 : PC_BP3H_MINB) k_bp3h(const BpArgs a)
{
    using namespace b3h;
    constexpr int N = 128, Q = 8, NW = N / 32;
    __shared__ __align__(16) float scratch[BP3H_WARPS][XSW];
    __shared__ uint8_t ubs[BP3H_WARPS][2][N];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane >> 4, l = lane & 15;
    const unsigned hm = 0xffffu << (16 * h);
    float *xs = &scratch[warp][HS * h];
    uint8_t *ub = ubs[warp][h];
    const BpLim lim = bp_lim<GMODE>(a.llr_max);
    const int base = 8 * l; // layout A: nodes base..base+7

    // frame-independent: the frozen prior R[0] and the CRC columns (layout A)
    const uint32_t fw = (__ldg(a.code.frozen_bits + (base >> 5)) >> (base & 31)) & 0xffu;
    float pri[Q];
    uint32_t col[Q];
#pragma unroll
    for (int r = 0; r < Q; ++r) {
        pri[r] = ((fw >> r) & 1u) ? bp_prior<GMODE>(lim) : bp_zero<GMODE>();
        col[r] = !RE && a.stop_mode == 0 ? __ldg(a.code.crc_cols + base + r) : 0u;
    }

    int f;
    if constexpr (PERS) {
        int t = 0;
        if (l == 0)
            t = atomicAdd(a.work, 1);
        f = __shfl_sync(hm, t, 0, 16);
    } else {
        f = 2 * (blockIdx.x * BP3H_WARPS + warp) + h;
    }
    if (f >= a.B)
        return;

    float Lch[Q]; // L[7], the channel row (layout C)
    float L1[Q], L2[Q], L3[Q], L4[Q], L5[Q], L6[Q];
    auto load_frame = [&](int fr) {
        const float *g = a.llr + (size_t)fr * N;
#pragma unroll
        for (int r = 0; r < Q; ++r)
            Lch[r] = bp_load<GMODE>(__ldg(g + xc(l, r)), a.llr_max);
#pragma unroll
        for (int r = 0; r < Q; ++r)
            L1[r] = L2[r] = L3[r] = L4[r] = L5[r] = L6[r] = bp_zero<GMODE>();
    };
    load_frame(f);

    float su[Q];
    float R1[Q], R2[Q], R3[Q], R3b[Q], R4[Q], R5[Q], R6[Q], R6c[Q];
    int it = 0;
    for (;;) {
        ++it;
        // ================= R sweep (R[7] is not needed) =================
        stage<GMODE, true, 1>(pri, L1, R1, lim);
        stage<GMODE, true, 2>(R1, L2, R2, lim);
        stage<GMODE, true, 4>(R2, L3, R3, lim);
        a_to_b(R3, R3b, xs, l, hm);
        stage<GMODE, true, 1>(R3b, L4, R4, lim);
        stage<GMODE, true, 2>(R4, L5, R5, lim);
        stage<GMODE, true, 4>(R5, L6, R6, lim);
        b_c<true>(R6, R6c, xs, l, hm);
        // ================= L sweep =================
        {
            float L6c[Q];
            stage<GMODE, false, 4>(R6c, Lch, L6c, lim);
            b_c<false>(L6c, L6, xs, l, hm);
        }
        stage<GMODE, false, 4>(R5, L6, L5, lim);
        stage<GMODE, false, 2>(R4, L5, L4, lim);
        {
            float L3b[Q];
            stage<GMODE, false, 1>(R3b, L4, L3b, lim);
            b_to_a(L3b, L3, xs, l, hm);
        }
        stage<GMODE, false, 4>(R2, L3, L2, lim);
        stage<GMODE, false, 2>(R1, L2, L1, lim);
#pragma unroll
        for (int r1 = 0; r1 < Q; r1 += 2) { // boundary 1: L[0], then soft_u = L[0] + R[0]
            const int r2 = r1 + 1;
            float o1, o2;
            bp_pe2<GMODE, false>(L1[r1], bp_comb<GMODE>(L1[r2], pri[r2]), pri[r1], L1[r2], lim, o1, o2);
            su[r1] = bp_comb<GMODE>(o1, pri[r1]);
            su[r2] = bp_comb<GMODE>(o2, pri[r2]);
        }
        // ================= stop rule (CRC; stop_mode 2 runs i_max iterations) =================
        bool stop = false;
        if (!RE && a.stop_mode == 0) {
            uint32_t syn = 0;
#pragma unroll
            for (int r = 0; r < Q; ++r)
                syn ^= bp_neg<GMODE>(su[r]) ? col[r] : 0u;
#pragma unroll
            for (int s = 8; s >= 1; s >>= 1)
                syn ^= __shfl_xor_sync(hm, syn, s, 16);
            stop = (syn == a.code.crc_offset);
        }
        if constexpr (RE) {
            // re-encode stop (bp.py:187), as in k_bp3: x_hat = hard(L[7] + R[7]) with
            // R[7] from boundary 7 of the R sweep (layout C, through the half's
            // decision bytes into layout A), against the polar transform of the
            // thread's 8 decisions: in registers, then across the half's lanes
            float R7[Q];
            stage<GMODE, true, 4>(R6c, Lch, R7, lim);
            __syncwarp(hm);
#pragma unroll
            for (int r = 0; r < Q; ++r)
                ub[xc(l, r)] = bp_neg<GMODE>(bp_comb<GMODE>(Lch[r], R7[r]));
            uint32_t v = 0;
#pragma unroll
            for (int r = 0; r < Q; ++r)
                v |= (bp_neg<GMODE>(su[r]) ? 1u : 0u) << r;
#pragma unroll
            for (int hh = 1; hh < Q; hh <<= 1)
                v ^= (v >> hh) & (hh == 1 ? 0x55u : (hh == 2 ? 0x33u : 0x0Fu));
#pragma unroll
            for (int s = 1; s < 16; s <<= 1) {
                const uint32_t pv = __shfl_xor_sync(hm, v, s, 16);
                if (!(l & s))
                    v ^= pv;
            }
            __syncwarp(hm);
            uint32_t xh = 0;
#pragma unroll
            for (int r = 0; r < Q; ++r)
                xh |= (uint32_t)ub[base + r] << r;
            stop = !__any_sync(hm, v != xh);
        }
        if (!stop && it < a.i_max)
            continue;

        // ---- outputs of frame f (as k_bp2 / k_bp3) ----
        if (l == 0) {
            if (a.t_done != nullptr)
                a.t_done[f] = globaltimer();
            a.iters[f] = stop ? it : a.i_max;
            a.conv[f] = stop ? 1 : 0;
        }
        __syncwarp(hm);
#pragma unroll
        for (int r = 0; r < Q; ++r)
            ub[base + r] = bp_neg<GMODE>(su[r]);
        if (a.soft_u != nullptr) {
#pragma unroll
            for (int r = 0; r < Q; r += 2)
                *reinterpret_cast<float2 *>(a.soft_u + (size_t)f * N + base + r) =
                    make_float2(bp_store<GMODE>(su[r]), bp_store<GMODE>(su[r + 1]));
        }
        if (a.soft_x != nullptr) {
            // soft_x = L[n] + R[n] (bp.py:164-168): boundary 7 of the R sweep, in layout C
            float R7[Q];
            stage<GMODE, true, 4>(R6c, Lch, R7, lim);
#pragma unroll
            for (int r = 0; r < Q; ++r)
                a.soft_x[(size_t)f * N + xc(l, r)] = bp_store<GMODE>(bp_comb<GMODE>(Lch[r], R7[r]));
        }
        __syncwarp(hm);
        // 16 decisions per ballot: words of 32 from two ballots of the half
        if (a.u_bits != nullptr) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const uint32_t lo = __ballot_sync(hm, ub[32 * w + l]) >> (16 * h);
                const uint32_t hi = __ballot_sync(hm, ub[32 * w + 16 + l]) >> (16 * h);
                if (l == 0)
                    a.u_bits[(size_t)f * NW + w] = lo | (hi << 16);
            }
        }
        if (a.payload != nullptr) {
            const int m = a.code.m, MW = (m + 31) >> 5;
            for (int w = 0; w < MW; ++w) {
                const int b0 = 32 * w + l, b1 = b0 + 16;
                const uint32_t lo = __ballot_sync(hm, b0 < m && ub[__ldg(a.code.info_pos + b0)]) >> (16 * h);
                const uint32_t hi = __ballot_sync(hm, b1 < m && ub[__ldg(a.code.info_pos + b1)]) >> (16 * h);
                if (l == 0)
                    a.payload[(size_t)f * MW + w] = lo | (hi << 16);
            }
        }
        if constexpr (!PERS)
            break;
        int t = 0;
        if (l == 0)
            t = atomicAdd(a.work, 1);
        f = __shfl_sync(hm, t, 0, 16);
        if (f >= a.B)
            break;
        load_frame(f);
        it = 0;
    }
}

bool bp3h_eligible(const BpArgs &a, int g_mode, int tpf)
{
    return a.code.n == 7 && (g_mode == 0 || g_mode == 1) && (tpf == 0 || tpf == 16);
}

template <int GMODE>
static int launch_bp3h_t(const BpArgs &a, cudaStream_t s)
{
    const bool pers = a.work != nullptr, re = a.stop_mode == 1;
    auto kern = pers ? (re ? k_bp3h<GMODE, true, true> : k_bp3h<GMODE, true, false>)
                     : (re ? k_bp3h<GMODE, false, true> : k_bp3h<GMODE, false, false>);
    const int per_cta = 2 * BP3H_WARPS;
    long long grid = ((long long)a.B + per_cta - 1) / per_cta;
    if (pers) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * BP3H_WARPS, 0) != cudaSuccess ||
            per_sm < 1)
            return PC_ERR_CUDA;
        if ((long long)sms * per_sm < grid)
            grid = (long long)sms * per_sm;
        if (cudaMemsetAsync(a.work, 0, sizeof(int32_t), s) != cudaSuccess)
            return PC_ERR_CUDA;
    }
    kern<<<(int)grid, 32 * BP3H_WARPS, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

int launch_bp3h(const BpArgs &a, int g_mode, cudaStream_t s)
{
    if (a.B == 0)
        return PC_OK;
    if (g_mode == 0)
        return launch_bp3h_t<0>(a, s);
    if (g_mode == 1)
        return launch_bp3h_t<1>(a, s);
    return PC_ERR_UNSUPPORTED;
}

} // namespace pc
