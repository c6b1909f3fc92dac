// bp.cu -- K1: belief-propagation decoding on the polar factor graph (sm_100a).
//
// Restates bp.py (reference /root/reference/pkg/src/polarsim/bp.py):
//   init_graph      bp.py:120-135   L[n] = clip(llr), R[0] = llr_max * frozen
//   iterate_once    bp.py:138-161   R sweep j = 1..n, L sweep j = n..1, in place
//   g_fn            bp.py:86-100    exact / min node update, clipped
//   stopping_check  bp.py:176-191   evaluated after EVERY iteration (bp.py:203-208)
//
// One CTA decodes one frame.  Shared memory holds the persistent message
// rows R[1..n-1] and L[1..n] in fp32 (R[0] is the frozen prior, recomputed
// from a bitmask; L[0] and R[n] are never read by a sweep, so L[0] only feeds
// the hard decisions and R[n] is produced once at exit for soft_x, unless the
// re-encode stop rule needs it every iteration).  Every boundary of a sweep
// is one parallel step over the N/2 processing elements followed by a CTA
// barrier; the CRC verdict is an XOR reduction of per-position syndrome
// columns over the decided ones (codes.py CodeConfig.crc_columns).
//
// The exact g is evaluated in the cancellation-free form
//     g(a, b) = sgn(a) sgn(b) [ m + sp(|a|+|b|) - sp(||a|-|b||) ],
//     m = min(|a|,|b|),  sp(x) = log1p(exp(-x)) = ln2 * lg2(1 + 2^(-x log2 e)),
// which equals logaddexp(0,a+b) - logaddexp(a,b) of bp.py:95 (4 MUFU ops).
// The magnitude is clamped to [0, m], the range the exact value lies in.
#include "args.cuh"
#include "bp_math.cuh"

namespace pc {


// One boundary of the R sweep (writes R[j]) or L sweep (writes L[j-1]).
// Rprev = R[j-1] (nullptr for j == 1: use the frozen prior), Lj = L[j].
template <int GMODE, bool RSWEEP>
__device__ __forceinline__ void bp_pe(int j, int p, const float *__restrict__ Rprev, const float *__restrict__ Lj,
                                      const uint32_t *frz, BpLim lim, float &o1, float &o2, float &av, float &r2)
{
    const int h = 1 << (j - 1);
    const int i1 = ((p >> (j - 1)) << j) | (p & (h - 1));
    const int i2 = i1 + h;
    if (Rprev == nullptr) {
        av = bit_of(frz, i1) ? bp_prior<GMODE>(lim) : bp_zero<GMODE>();
        r2 = bit_of(frz, i2) ? bp_prior<GMODE>(lim) : bp_zero<GMODE>();
    } else {
        av = Rprev[i1];
        r2 = Rprev[i2];
    }
    const float l1 = Lj[i1], l2 = Lj[i2];
    if (RSWEEP)
        bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2), l1, r2, lim, o1, o2);
    else
        bp_pe2<GMODE, false>(l1, bp_comb<GMODE>(l2, r2), av, l2, lim, o1, o2);
}

template <int LOGN>
__device__ __forceinline__ void pe_nodes(int j, int p, int &i1, int &i2)
{
    const int h = 1 << (j - 1);
    i1 = ((p >> (j - 1)) << j) | (p & (h - 1));
    i2 = i1 + h;
}

template <int LOGN, int TPF, int GMODE>
__global__ void __launch_bounds__(TPF) k_bp_decode(const BpArgs a)
{
    constexpr int N = 1 << LOGN;
    constexpr int NPE = N / 2;
    constexpr int PPT = NPE / TPF; // processing elements per thread per boundary
    constexpr int NW = (N + 31) / 32;
    constexpr int NWARP = (TPF + 31) / 32;
    constexpr uint32_t FULL = TPF >= 32 ? 0xffffffffu : ((1u << TPF) - 1u);
    static_assert(PPT >= 1 && PPT * TPF == NPE, "TPF must divide N/2");

    extern __shared__ __align__(16) float sm[];
    float *Rs = sm;                   // R[1..n-1]
    float *Ls = sm + (LOGN - 1) * N;  // L[1..n]
    float *Rn = Ls + LOGN * N;        // R[n] (re-encode stop only)
    uint8_t *ub = reinterpret_cast<uint8_t *>(Rn + (a.stop_mode == 1 ? N : 0));
    __shared__ uint32_t frz[NW];
    __shared__ uint32_t red[NWARP];

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int f = blockIdx.x;
    const BpLim lim = bp_lim<GMODE>(a.llr_max); // clip bounds in the mode's message domain (bp_math.cuh)

    for (int w = tid; w < NW; w += TPF)
        frz[w] = a.code.frozen_bits[w];
    const float *x = a.llr + (size_t)f * N;
    float *Lch = Ls + (LOGN - 1) * N;
    for (int i = tid; i < N; i += TPF)
        Lch[i] = bp_load<GMODE>(__ldg(x + i), a.llr_max);
    for (int i = tid; i < (LOGN - 1) * N; i += TPF) {
        Rs[i] = bp_zero<GMODE>();
        Ls[i] = bp_zero<GMODE>();
    }
    // CRC columns of the two nodes each boundary-1 element decides.
    uint32_t col[PPT][2];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const int p = tid + q * TPF;
        col[q][0] = a.stop_mode == 0 ? __ldg(a.code.crc_cols + 2 * p) : 0u;
        col[q][1] = a.stop_mode == 0 ? __ldg(a.code.crc_cols + 2 * p + 1) : 0u;
    }
    __syncthreads();

    float su[PPT][2];
    int it = 0;
    bool stop = false;
    for (;;) {
        ++it;
        // ---- R sweep: boundaries 1..n (R[n] only when re-encoding) ----
#pragma unroll
        for (int j = 1; j <= LOGN; ++j) {
            if (j == LOGN && a.stop_mode != 1)
                break;
            const float *Rp = (j == 1) ? nullptr : Rs + (j - 2) * N;
            float *Rd = (j == LOGN) ? Rn : Rs + (j - 1) * N;
            const float *Lj = Ls + (j - 1) * N;
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                const int p = tid + q * TPF;
                float o1, o2, av, r2;
                bp_pe<GMODE, true>(j, p, Rp, Lj, frz, lim, o1, o2, av, r2);
                int i1, i2;
                pe_nodes<LOGN>(j, p, i1, i2);
                Rd[i1] = o1;
                Rd[i2] = o2;
            }
            __syncthreads();
        }
        // ---- L sweep: boundaries n..1 ----
#pragma unroll
        for (int j = LOGN; j >= 1; --j) {
            const float *Rp = (j == 1) ? nullptr : Rs + (j - 2) * N;
            const float *Lj = Ls + (j - 1) * N;
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                const int p = tid + q * TPF;
                float o1, o2, av, r2;
                bp_pe<GMODE, false>(j, p, Rp, Lj, frz, lim, o1, o2, av, r2);
                if (j > 1) {
                    int i1, i2;
                    pe_nodes<LOGN>(j, p, i1, i2);
                    Ls[(j - 2) * N + i1] = o1;
                    Ls[(j - 2) * N + i2] = o2;
                } else {
                    su[q][0] = bp_comb<GMODE>(o1, av); // soft_u = L[0] + R[0] on nodes 2p, 2p+1
                    su[q][1] = bp_comb<GMODE>(o2, r2);
                }
            }
            if (j > 1)
                __syncthreads();
        }
        // ---- stop rule ----
        if (a.stop_mode == 0) {
            uint32_t syn = 0;
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                syn ^= bp_neg<GMODE>(su[q][0]) ? col[q][0] : 0u;
                syn ^= bp_neg<GMODE>(su[q][1]) ? col[q][1] : 0u;
            }
            syn = __reduce_xor_sync(FULL, syn);
            if (lane == 0)
                red[warp] = syn;
            __syncthreads();
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < NWARP; ++w)
                tot ^= red[w];
            stop = (tot == a.code.crc_offset);
        } else if (a.stop_mode == 1) {
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                const int p = tid + q * TPF;
                ub[2 * p] = bp_neg<GMODE>(su[q][0]);
                ub[2 * p + 1] = bp_neg<GMODE>(su[q][1]);
            }
            __syncthreads();
            for (int h = 1; h < N; h <<= 1) { // polar_transform on the byte vector
                for (int e = tid; e < NPE; e += TPF) {
                    const int i1 = ((e / h) * 2 * h) + (e % h);
                    ub[i1] ^= ub[i1 + h];
                }
                __syncthreads();
            }
            int bad = 0;
            for (int i = tid; i < N; i += TPF)
                bad |= ub[i] != (uint8_t)bp_neg<GMODE>(bp_comb<GMODE>(Lch[i], Rn[i]));
            stop = !__syncthreads_or(bad);
        } else {
            __syncthreads();
        }
        if (stop || it >= a.i_max)
            break;
    }

    // ---- outputs ----
    if (a.t_done != nullptr && tid == 0)
        a.t_done[f] = globaltimer();
    if (tid == 0) {
        a.iters[f] = stop ? it : a.i_max;
        a.conv[f] = stop ? 1 : 0;
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        const int p = tid + q * TPF;
        if (a.soft_u != nullptr)
            *reinterpret_cast<float2 *>(a.soft_u + (size_t)f * N + 2 * p) =
                make_float2(bp_store<GMODE>(su[q][0]), bp_store<GMODE>(su[q][1]));
        ub[2 * p] = bp_neg<GMODE>(su[q][0]);
        ub[2 * p + 1] = bp_neg<GMODE>(su[q][1]);
    }
    if (a.soft_x != nullptr) {
        // R[n] from the final R[n-1] and L[n] (R[n] is not read by the sweeps).
        const float *Rp = (LOGN == 1) ? nullptr : Rs + (LOGN - 2) * N;
        for (int p = tid; p < NPE; p += TPF) {
            float o1, o2, av, r2;
            bp_pe<GMODE, true>(LOGN, p, Rp, Lch, frz, lim, o1, o2, av, r2);
            int i1, i2;
            pe_nodes<LOGN>(LOGN, p, i1, i2);
            a.soft_x[(size_t)f * N + i1] = bp_store<GMODE>(bp_comb<GMODE>(Lch[i1], o1));
            a.soft_x[(size_t)f * N + i2] = bp_store<GMODE>(bp_comb<GMODE>(Lch[i2], o2));
        }
    }
    __syncthreads();
    if (a.u_bits != nullptr)
        for (int w = tid; w < NW; w += TPF) {
            uint32_t v = 0;
            for (int b = 0; b < 32 && 32 * w + b < N; ++b)
                v |= (uint32_t)ub[32 * w + b] << b;
            a.u_bits[(size_t)f * NW + w] = v;
        }
    if (a.payload != nullptr) {
        const int MW = (a.code.m + 31) >> 5;
        for (int w = tid; w < MW; w += TPF) {
            uint32_t v = 0;
            for (int b = 0; b < 32 && 32 * w + b < a.code.m; ++b)
                v |= (uint32_t)ub[__ldg(a.code.info_pos + 32 * w + b)] << b;
            a.payload[(size_t)f * MW + w] = v;
        }
    }
}

// Teacher-forced hook: one full iterate_once on explicit [B][n+1][N] state.
// SMEM = true stages the frame's state in shared memory (N <= 2048); for
// N = 4096 (426 KB of state) the same sweeps run in place on global memory.
template <int GMODE, bool SMEM>
__global__ void k_bp_iterate(float *l_msgs, float *r_msgs, int n, float llr_max)
{
    extern __shared__ __align__(16) float st[];
    const int N = 1 << n;
    const size_t base = (size_t)blockIdx.x * (n + 1) * N;
    constexpr float KIN = bp_unit_in<GMODE>();
    float *L = SMEM ? st : l_msgs + base;
    float *R = SMEM ? st + (size_t)(n + 1) * N : r_msgs + base;
    const float lim_out = llr_max;
    const BpLim lim = bp_lim<GMODE>(llr_max);
    for (int i = threadIdx.x; i < (n + 1) * N; i += blockDim.x) { // into the mode's message domain
        const float l = l_msgs[base + i] * KIN, r = r_msgs[base + i] * KIN;
        L[i] = GMODE == 0 ? ex2_approx(l) : l;
        R[i] = GMODE == 0 ? ex2_approx(r) : r;
    }
    __syncthreads();
    const int NPE = N / 2;
    for (int j = 1; j <= n; ++j) {
        const int h = 1 << (j - 1);
        for (int p = threadIdx.x; p < NPE; p += blockDim.x) {
            const int i1 = ((p >> (j - 1)) << j) | (p & (h - 1)), i2 = i1 + h;
            const float av = R[(j - 1) * N + i1], r2 = R[(j - 1) * N + i2];
            const float l1 = L[j * N + i1], l2 = L[j * N + i2];
            float o1, o2;
            bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2), l1, r2, lim, o1, o2);
            R[j * N + i1] = o1;
            R[j * N + i2] = o2;
        }
        __syncthreads();
    }
    for (int j = n; j >= 1; --j) {
        const int h = 1 << (j - 1);
        for (int p = threadIdx.x; p < NPE; p += blockDim.x) {
            const int i1 = ((p >> (j - 1)) << j) | (p & (h - 1)), i2 = i1 + h;
            const float av = R[(j - 1) * N + i1], r2 = R[(j - 1) * N + i2];
            const float l1 = L[j * N + i1], l2 = L[j * N + i2];
            float o1, o2;
            bp_pe2<GMODE, false>(l1, bp_comb<GMODE>(l2, r2), av, l2, lim, o1, o2);
            L[(j - 1) * N + i1] = o1;
            L[(j - 1) * N + i2] = o2;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < (n + 1) * N; i += blockDim.x) {
        l_msgs[base + i] = clampf(bp_store<GMODE>(L[i]), lim_out);
        r_msgs[base + i] = clampf(bp_store<GMODE>(R[i]), lim_out);
    }
}

// ------------------------------------------------------------- launchers --

static size_t bp_smem_bytes(int logn, int stop_mode)
{
    const size_t N = (size_t)1 << logn;
    return ((size_t)(2 * logn - 1) + (stop_mode == 1 ? 1 : 0)) * N * sizeof(float) + N;
}

template <int LOGN, int TPF, int GMODE>
static int launch_bp_t(const BpArgs &a, cudaStream_t s)
{
    auto kern = k_bp_decode<LOGN, TPF, GMODE>;
    const size_t smem = bp_smem_bytes(LOGN, a.stop_mode);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return PC_ERR_CUDA;
    kern<<<a.B, TPF, smem, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

template <int LOGN, int GMODE>
static int launch_bp_n(const BpArgs &a, int tpf, cudaStream_t s)
{
    constexpr int NPE = (1 << LOGN) / 2;
    if constexpr (NPE <= 32) {
        return launch_bp_t<LOGN, NPE, GMODE>(a, s);
    } else {
        if (tpf <= 0)
            tpf = NPE >= 256 ? 256 : NPE;
        if (tpf > NPE)
            tpf = NPE;
        switch (tpf) {
        case 32: return launch_bp_t<LOGN, 32, GMODE>(a, s);
        case 64: return launch_bp_t<LOGN, (NPE >= 64 ? 64 : NPE), GMODE>(a, s);
        case 128: return launch_bp_t<LOGN, (NPE >= 128 ? 128 : NPE), GMODE>(a, s);
        case 256: return launch_bp_t<LOGN, (NPE >= 256 ? 256 : NPE), GMODE>(a, s);
        case 512: return launch_bp_t<LOGN, (NPE >= 512 ? 512 : NPE), GMODE>(a, s);
        case 1024: return launch_bp_t<LOGN, (NPE >= 1024 ? 1024 : NPE), GMODE>(a, s);
        default: return PC_ERR_UNSUPPORTED;
        }
    }
}

template <int GMODE>
static int launch_bp_g(const BpArgs &a, int logn, int tpf, cudaStream_t s)
{
    switch (logn) {
    case 1: return launch_bp_n<1, GMODE>(a, tpf, s);
    case 2: return launch_bp_n<2, GMODE>(a, tpf, s);
    case 3: return launch_bp_n<3, GMODE>(a, tpf, s);
    case 4: return launch_bp_n<4, GMODE>(a, tpf, s);
    case 5: return launch_bp_n<5, GMODE>(a, tpf, s);
    case 6: return launch_bp_n<6, GMODE>(a, tpf, s);
    case 7: return launch_bp_n<7, GMODE>(a, tpf, s);
    case 8: return launch_bp_n<8, GMODE>(a, tpf, s);
    case 9: return launch_bp_n<9, GMODE>(a, tpf, s);
    case 10: return launch_bp_n<10, GMODE>(a, tpf, s);
    case 11: return launch_bp_n<11, GMODE>(a, tpf, s);
    default: return PC_ERR_UNSUPPORTED;
    }
}

int launch_bp_decode(const BpArgs &a, int g_mode, int tpf, int kernel, cudaStream_t s)
{
    if (a.B == 0)
        return PC_OK;
    if (g_mode == 2 || g_mode == 3) // exact g, per-g / round-1 log-domain forms: K1 v2 only
        return launch_bp2(a, g_mode, tpf, s);
    // kernel: 0 auto (v3 where eligible, else v2, else v1), 1 v1, 2 v2, 3 v3
    if (kernel == 3) {
        if (bp3h_eligible(a, g_mode, tpf))
            return launch_bp3h(a, g_mode, s);
        return bp3_eligible(a, g_mode, tpf) ? launch_bp3(a, g_mode, s) : PC_ERR_UNSUPPORTED;
    }
    if (kernel == 0 && bp3h_eligible(a, g_mode, tpf))
        return launch_bp3h(a, g_mode, s);
    if (kernel == 0 && bp3_eligible(a, g_mode, tpf))
        return launch_bp3(a, g_mode, s);
    if (kernel == 2 && !bp2_eligible(a, g_mode, tpf))
        return PC_ERR_UNSUPPORTED;
    if (kernel != 1 && bp2_eligible(a, g_mode, tpf))
        return launch_bp2(a, g_mode, tpf, s);
    return g_mode == 0 ? launch_bp_g<0>(a, a.code.n, tpf, s) : launch_bp_g<1>(a, a.code.n, tpf, s);
}

int launch_bp_iterate(float *l, float *r, int B, int n, int g_mode, float lim, cudaStream_t s)
{
    if (B == 0)
        return PC_OK;
    const size_t smem = (size_t)2 * (n + 1) * ((size_t)1 << n) * sizeof(float);
    const int threads = (1 << (n - 1)) >= 256 ? 256 : (1 << (n - 1));
    if (smem > 200 * 1024) {
        auto kern = g_mode == 0 ? k_bp_iterate<0, false> : (g_mode == 1 ? k_bp_iterate<1, false> : k_bp_iterate<3, false>);
        kern<<<B, threads, 0, s>>>(l, r, n, lim);
        return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
    }
    auto kern = g_mode == 0 ? k_bp_iterate<0, true> : (g_mode == 1 ? k_bp_iterate<1, true> : k_bp_iterate<3, true>);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return PC_ERR_CUDA;
    kern<<<B, threads, smem, s>>>(l, r, n, lim);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

} // namespace pc
