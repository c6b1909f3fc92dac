// bp3.cu -- K1 v3: BP decoding with warp-local stages in three register
// layouts joined by warp-private shared-memory transposes (sm_100a).
//
// Same recursion, stop rules and outputs as k_bp2 (bp2.cu; reference
// bp.py:120-217) and the same per-PE arithmetic (bp_math.cuh::bp_pe2), so the
// two kernels give bit-identical iterations, decisions and soft values.  What
// changes is how the warp-local boundaries 1..8 are mapped.  A thread owns
// Q = 8 nodes of its warp's 256 and keeps them in registers in one of three
// layouts (x = warp-local node, l = lane, r = register):
//   A  x = 8l + r                      boundaries 1, 2, 3 (strides 1, 2, 4)
//   B  x = (l & 7) + 8r + 64(l >> 3)   boundaries 4, 5, 6 (strides 8, 16, 32)
//   C  x = l + 32(r >> 2) + 64(r & 3)  boundaries 7, 8    (strides 64, 128)
// Every warp-local boundary is then a butterfly between registers of one
// thread: no shuffles and none of the lane-role selects that k_bp2's
// lane-pair exchange needs (ncu, k_bp2 TPF=128: FSEL 20% and SHFL 7% of all
// instructions).  A row crosses layouts once per sweep through 280 floats of
// warp-private shared memory: R[3] A->B and R[6] B->C in the R sweep, L[6]
// C->B and L[3] B->A in the L sweep.  The scratch index x + 8(x >> 6) makes the
// scalar B and C accesses conflict-free (banks (l & 7) + 8(l >> 3) + 8r and
// l + 8r'); A uses 16-byte accesses.  Boundaries above 8 run in shared memory
// in radix-4 pairs exactly as in k_bp2.
#include "args.cuh"
#include "bp_math.cuh"

namespace pc {

namespace b3 {

constexpr int XSW = 280; // warp scratch floats (256 nodes + 3 x 8 padding)

__device__ __forceinline__ int xa(int l, int r) { return 8 * l + r; }
__device__ __forceinline__ int xb(int l, int r) { return (l & 7) + 8 * r + 64 * (l >> 3); }
__device__ __forceinline__ int xc(int l, int r) { return l + 32 * (r >> 2) + 64 * (r & 3); }
__device__ __forceinline__ int xpad(int x) { return x + ((x >> 6) << 3); }

// One warp-local boundary inside a thread: register pairs (r, r + H).
// R sweep: out = R[j] from Rp = R[j-1], Lj = L[j]; L sweep: out = L[j-1].
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

// Layout transposes through the warp scratch xs.  The leading __syncwarp
// orders the writes after every lane's reads of the previous transpose.
__device__ __forceinline__ void a_to_b(const float (&v)[8], float (&o)[8], float *xs, int l)
{
    __syncwarp();
    float *p = xs + xpad(xa(l, 0)); // 32-byte aligned: 8l + 8(l >> 3)
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4 *>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 8; ++r)
        o[r] = xs[xpad(xb(l, r))];
}

__device__ __forceinline__ void b_to_a(const float (&v)[8], float (&o)[8], float *xs, int l)
{
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 8; ++r)
        xs[xpad(xb(l, r))] = v[r];
    __syncwarp();
    const float *p = xs + xpad(xa(l, 0));
    const float4 u = *reinterpret_cast<const float4 *>(p), w = *reinterpret_cast<const float4 *>(p + 4);
    o[0] = u.x, o[1] = u.y, o[2] = u.z, o[3] = u.w, o[4] = w.x, o[5] = w.y, o[6] = w.z, o[7] = w.w;
}

template <bool B2C>
__device__ __forceinline__ void b_c(const float (&v)[8], float (&o)[8], float *xs, int l)
{
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 8; ++r)
        xs[xpad(B2C ? xb(l, r) : xc(l, r))] = v[r];
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 8; ++r)
        o[r] = xs[xpad(B2C ? xc(l, r) : xb(l, r))];
}

} // namespace b3

#ifndef PC_BP3_MINB12
#define PC_BP3_MINB12 1 // N = 4096: the one CTA per SM may use up to 128 registers (119; +0.6%)
#endif
#ifndef PC_BP3_MINB10
#define PC_BP3_MINB10 5 // N = 1024: 5 CTAs per SM (96 registers; +0.7% over the compiler's own choice)
#endif
#ifndef PC_BP3_FUSE
#define PC_BP3_FUSE 1
#endif

__host__ __device__ constexpr int bp3_smem_floats(int logn)
{
    // R[8..n-1], L[8..n], N bytes of decisions, warp scratch
    return (2 * (logn - 8) + 1) * (1 << logn) + (1 << logn) / 4 + ((1 << logn) / 256) * b3::XSW;
}

template <int LOGN, int GMODE, bool RE, bool PERS>
__global__ void __launch_bounds__((1 << LOGN) / 8, (LOGN == 10 && GMODE == 0) ? PC_BP3_MINB10
                                                   : ((LOGN == 12 && GMODE == 0) ? PC_BP3_MINB12 : 0)) k_bp3(const BpArgs a)
{
    using namespace b3;
    constexpr int N = 1 << LOGN;
    constexpr int TPF = N / 8;
    constexpr int Q = 8;
    constexpr int BW = 8;              // warp-local boundaries 1..8
    constexpr int NSR = LOGN - BW;     // shared R rows: R[8..n-1]
    constexpr int NSL = LOGN - BW + 1; // shared L rows: L[8..n]
    constexpr int NW = N / 32;
    constexpr int NWARP = TPF / 32;
    constexpr int PPT = N / 2 / TPF;   // shared-memory PEs per thread (single boundaries)
    // fused turn of the sweeps at the top pair (n-1, n) when the shared
    // boundaries 9..n pair up evenly (N = 1024, 4096)
    constexpr bool FUSE = LOGN >= BW + 2 && (LOGN - BW) % 2 == 0 && PC_BP3_FUSE;
    constexpr int RTOP = FUSE ? LOGN - 2 : LOGN - 1; // highest R row of the R sweep proper
    static_assert(LOGN >= 8 && LOGN <= 12, "bp3 geometry: 256..4096 nodes, 8 per thread");

    extern __shared__ __align__(16) float sm[];
    float *Rs = sm;
    float *Ls = sm + NSR * N;
    uint8_t *ub = reinterpret_cast<uint8_t *>(Ls + NSL * N);
    __shared__ uint32_t frz[NW];
    __shared__ uint32_t red[NWARP];
    __shared__ uint32_t xw[RE ? TPF : 1];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float *xs = Ls + NSL * N + N / 4 + warp * XSW;
    int f = blockIdx.x;
    const BpLim lim = bp_lim<GMODE>(a.llr_max);
    const int wb = warp * 256;
    const int base = wb + 8 * lane; // layout A: the thread's nodes base..base+7

    __shared__ __align__(8) uint64_t ch_bar;
    float *Lch = Ls + (NSL - 1) * N;
    __shared__ int next_f;
    if (tid == 0) {
        mbar_init(&ch_bar, 1);
        if constexpr (PERS)
            next_f = atomicAdd(a.work, 1);
    }
    for (int w = tid; w < NW; w += TPF)
        frz[w] = a.code.frozen_bits[w];
    __syncthreads();
    if constexpr (PERS)
        f = next_f;
    uint32_t phase = 0;
    while (f < a.B) {
    if (tid == 0)
        tma_load_1d(Lch, a.llr + (size_t)f * N, N * sizeof(float), &ch_bar);
    for (int i = tid; i < (NSL - 1) * N; i += TPF)
        Ls[i] = bp_zero<GMODE>();
    mbar_wait(&ch_bar, phase);
    phase ^= 1u;
    for (int i = 4 * tid; i < N; i += 4 * TPF) {
        const float4 v = *reinterpret_cast<const float4 *>(Lch + i);
        *reinterpret_cast<float4 *>(Lch + i) = make_float4(bp_load<GMODE>(v.x, a.llr_max), bp_load<GMODE>(v.y, a.llr_max),
                                                          bp_load<GMODE>(v.z, a.llr_max), bp_load<GMODE>(v.w, a.llr_max));
    }
    // L rows kept across iterations: L[1..3] in layout A, L[4..6] in B, L[7] in C
    float L1[Q], L2[Q], L3[Q], L4[Q], L5[Q], L6[Q], L7[Q];
#pragma unroll
    for (int r = 0; r < Q; ++r)
        L1[r] = L2[r] = L3[r] = L4[r] = L5[r] = L6[r] = L7[r] = bp_zero<GMODE>();
    uint32_t col[Q];
#pragma unroll
    for (int r = 0; r < Q; ++r)
        col[r] = a.stop_mode == 0 ? __ldg(a.code.crc_cols + base + r) : 0u;
    __syncthreads();
    const uint32_t fw = frz[base >> 5] >> (base & 31);
    float pri[Q]; // R[0]: the frozen prior (layout A)
#pragma unroll
    for (int r = 0; r < Q; ++r)
        pri[r] = ((fw >> r) & 1u) ? bp_prior<GMODE>(lim) : bp_zero<GMODE>();

    float su[Q];
    int it = 0;
    bool stop = false;
    float R1[Q], R2[Q], R3[Q], R3b[Q], R4[Q], R5[Q], R6[Q], R6c[Q], R7[Q]; // rewritten by every R sweep
    for (;;) {
        ++it;
        // ================= R sweep =================
        stage<GMODE, true, 1>(pri, L1, R1, lim);
        stage<GMODE, true, 2>(R1, L2, R2, lim);
        stage<GMODE, true, 4>(R2, L3, R3, lim);
        a_to_b(R3, R3b, xs, lane);
        stage<GMODE, true, 1>(R3b, L4, R4, lim);
        stage<GMODE, true, 2>(R4, L5, R5, lim);
        stage<GMODE, true, 4>(R5, L6, R6, lim);
        b_c<true>(R6, R6c, xs, lane);
        stage<GMODE, true, 1>(R6c, L7, R7, lim);
        if constexpr (LOGN > BW) { // boundary 8 writes R[8] (shared) for boundary 9
            float L8[Q], R8[Q];
#pragma unroll
            for (int r = 0; r < Q; ++r)
                L8[r] = Ls[wb + xc(lane, r)];
            stage<GMODE, true, 2>(R7, L8, R8, lim);
#pragma unroll
            for (int r = 0; r < Q; ++r)
                Rs[wb + xc(lane, r)] = R8[r];
        }
        __syncthreads();
        // shared-memory boundaries in radix-4 pairs (j, j+1), as in k_bp2; with
        // FUSE the top pair (n-1, n) is left to the fused turn below
#pragma unroll
        for (int j = BW + 1; j <= RTOP; j += 2) {
            const int h = 1 << (j - 1);
            const float *Rp = Rs + (j - 1 - BW) * N;
            float *Rd = Rs + (j - BW) * N;
            const float *Lj = Ls + (j - BW) * N;
            if (j + 1 <= RTOP) {
                float *Rd2 = Rs + (j + 1 - BW) * N;
                const float *Lj2 = Ls + (j + 1 - BW) * N;
#pragma unroll
                for (int q = 0; q < Q / 4; ++q) {
                    const int g = tid + q * TPF;
                    const int n0 = ((g >> (j - 1)) << (j + 1)) | (g & (h - 1));
                    const int n1 = n0 + h, n2 = n0 + 2 * h, n3 = n0 + 3 * h;
                    float o[4];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int i1 = e ? n2 : n0, i2 = i1 + h;
                        const float av = Rp[i1], r2v = Rp[i2], l1 = Lj[i1], l2 = Lj[i2];
                        bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, o[2 * e], o[2 * e + 1]);
                    }
                    Rd[n0] = o[0];
                    Rd[n1] = o[1];
                    Rd[n2] = o[2];
                    Rd[n3] = o[3];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int i1 = e ? n1 : n0, i2 = i1 + 2 * h;
                        const float av = o[e], r2v = o[e + 2], l1 = Lj2[i1], l2 = Lj2[i2];
                        float p1, p2;
                        bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, p1, p2);
                        Rd2[i1] = p1;
                        Rd2[i2] = p2;
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < PPT; ++q) {
                    const int p = tid + q * TPF;
                    const int i1 = ((p >> (j - 1)) << j) | (p & (h - 1)), i2 = i1 + h;
                    const float av = Rp[i1], r2v = Rp[i2], l1 = Lj[i1], l2 = Lj[i2];
                    float o1, o2;
                    bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, o1, o2);
                    Rd[i1] = o1;
                    Rd[i2] = o2;
                }
            }
            __syncthreads();
        }
        if constexpr (FUSE) {
            // The turn of the sweep: R[n-1] (boundary n-1), then L[n-1] (boundary
            // n) and L[n-2] (boundary n-1), group by group.  A radix-4 group
            // {g, g+h, g+2h, g+3h} (h = N/4) is closed under boundaries n-1 and n,
            // so R[n-1] stays in registers and no barrier separates the sweeps.
            // The operations and their inputs are those of the separate R single
            // and L pair passes (bit-identical).
            constexpr int j = LOGN - 1;
            constexpr int h = 1 << (j - 1);
            const float *Rp = Rs + (j - 1 - BW) * N;
            float *Rj = Rs + (j - BW) * N;
            float *Lm = Ls + (j - BW) * N;
            const float *Lt = Ls + (j + 1 - BW) * N;
            float *Ld = Ls + (j - 1 - BW) * N;
            const bool keep_r = RE || a.soft_x != nullptr; // R[n-1] is read after the loop
#pragma unroll 1
            for (int q = 0; q < Q / 4; ++q) {
                const int n0 = tid + q * TPF, n1 = n0 + h, n2 = n0 + 2 * h, n3 = n0 + 3 * h;
                float o[4], m[4], rp[4];
                rp[0] = Rp[n0];
                rp[1] = Rp[n1];
                rp[2] = Rp[n2];
                rp[3] = Rp[n3];
#pragma unroll
                for (int e = 0; e < 2; ++e) { // R[n-1] from R[n-2] and L[n-1] (old)
                    const float l1 = Lm[e ? n2 : n0], l2 = Lm[e ? n3 : n1];
                    bp_pe2<GMODE, true>(rp[2 * e], bp_comb<GMODE>(l2, rp[2 * e + 1]), l1, rp[2 * e + 1], lim, o[2 * e],
                                        o[2 * e + 1]);
                }
                if (keep_r) {
                    Rj[n0] = o[0];
                    Rj[n1] = o[1];
                    Rj[n2] = o[2];
                    Rj[n3] = o[3];
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) { // L[n-1] from the channel row and R[n-1]
                    const int i1 = e ? n1 : n0, i2 = i1 + 2 * h;
                    const float l1 = Lt[i1], l2 = Lt[i2];
                    bp_pe2<GMODE, false>(l1, bp_comb<GMODE>(l2, o[e + 2]), o[e], l2, lim, m[e], m[e + 2]);
                }
                Lm[n0] = m[0];
                Lm[n1] = m[1];
                Lm[n2] = m[2];
                Lm[n3] = m[3];
#pragma unroll
                for (int e = 0; e < 2; ++e) { // L[n-2] from L[n-1] and R[n-2]
                    const int i1 = e ? n2 : n0, i2 = i1 + h;
                    float o1, o2;
                    bp_pe2<GMODE, false>(m[2 * e], bp_comb<GMODE>(m[2 * e + 1], rp[2 * e + 1]), rp[2 * e],
                                         m[2 * e + 1], lim, o1, o2);
                    Ld[i1] = o1;
                    Ld[i2] = o2;
                }
            }
            __syncthreads();
        }
        // ================= L sweep =================
#pragma unroll
        for (int jt = FUSE ? LOGN - 2 : LOGN; jt >= BW + 1; jt -= 2) {
            if (jt - 1 >= BW + 1) {
                const int j = jt - 1;
                const int h = 1 << (j - 1);
                const float *Rj = Rs + (j - BW) * N;
                const float *Rp = Rs + (j - 1 - BW) * N;
                const float *Lt = Ls + (j + 1 - BW) * N;
                float *Lm = Ls + (j - BW) * N;
                float *Ld = Ls + (j - 1 - BW) * N;
#pragma unroll
                for (int q = 0; q < Q / 4; ++q) {
                    const int g = tid + q * TPF;
                    const int n0 = ((g >> (j - 1)) << (j + 1)) | (g & (h - 1));
                    const int n1 = n0 + h, n2 = n0 + 2 * h, n3 = n0 + 3 * h;
                    float m[4];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int i1 = e ? n1 : n0, i2 = i1 + 2 * h;
                        const float av = Rj[i1], r2v = Rj[i2], l1 = Lt[i1], l2 = Lt[i2];
                        float o1, o2;
                        bp_pe2<GMODE, false>(l1, bp_comb<GMODE>(l2, r2v), av, l2, lim, o1, o2);
                        m[e] = o1;
                        m[e + 2] = o2;
                    }
                    Lm[n0] = m[0];
                    Lm[n1] = m[1];
                    Lm[n2] = m[2];
                    Lm[n3] = m[3];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int i1 = e ? n2 : n0, i2 = i1 + h;
                        const float av = Rp[i1], r2v = Rp[i2], l1 = m[2 * e], l2 = m[2 * e + 1];
                        float o1, o2;
                        bp_pe2<GMODE, false>(l1, bp_comb<GMODE>(l2, r2v), av, l2, lim, o1, o2);
                        Ld[i1] = o1;
                        Ld[i2] = o2;
                    }
                }
            } else {
                const int j = jt;
                const int h = 1 << (j - 1);
                const float *Rp = Rs + (j - 1 - BW) * N;
                const float *Lj = Ls + (j - BW) * N;
                float *Ld = Ls + (j - 1 - BW) * N;
#pragma unroll
                for (int q = 0; q < PPT; ++q) {
                    const int p = tid + q * TPF;
                    const int i1 = ((p >> (j - 1)) << j) | (p & (h - 1)), i2 = i1 + h;
                    const float av = Rp[i1], r2v = Rp[i2], l1 = Lj[i1], l2 = Lj[i2];
                    float o1, o2;
                    bp_pe2<GMODE, false>(l1, bp_comb<GMODE>(l2, r2v), av, l2, lim, o1, o2);
                    Ld[i1] = o1;
                    Ld[i2] = o2;
                }
            }
            __syncthreads();
        }
        {
            // boundaries 8 and 7 in layout C (L[8] from shared memory: the channel row at N = 256)
            float L8[Q], L7n[Q], L6c[Q];
#pragma unroll
            for (int r = 0; r < Q; ++r)
                L8[r] = Ls[wb + xc(lane, r)];
            stage<GMODE, false, 2>(R7, L8, L7n, lim);
            stage<GMODE, false, 1>(R6c, L7n, L6c, lim);
#pragma unroll
            for (int r = 0; r < Q; ++r)
                L7[r] = L7n[r];
            b_c<false>(L6c, L6, xs, lane);
        }
        stage<GMODE, false, 4>(R5, L6, L5, lim);
        stage<GMODE, false, 2>(R4, L5, L4, lim);
        {
            float L3b[Q];
            stage<GMODE, false, 1>(R3b, L4, L3b, lim);
            b_to_a(L3b, L3, xs, lane);
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
        // ================= stop rule =================
        if (!RE && a.stop_mode == 0) {
            uint32_t syn = 0;
#pragma unroll
            for (int r = 0; r < Q; ++r)
                syn ^= bp_neg<GMODE>(su[r]) ? col[r] : 0u;
            syn = __reduce_xor_sync(0xffffffffu, syn);
            if (lane == 0)
                red[warp] = syn;
            __syncthreads();
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < NWARP; ++w)
                tot ^= red[w];
            stop = (tot == a.code.crc_offset);
        }
        if constexpr (RE && LOGN - 1 >= BW) {
            // re-encode stop (bp.py:187), as in k_bp2: R[n] from this iteration's R[n-1]
            const float *Rp = Rs + (LOGN - 1 - BW) * N;
#pragma unroll 1
            for (int p = tid; p < N / 2; p += TPF) {
                const int i1 = p, i2 = p + N / 2;
                float o1, o2;
                bp_pe2<GMODE, true>(Rp[i1], bp_comb<GMODE>(Lch[i2], Rp[i2]), Lch[i1], Rp[i2], lim, o1, o2);
                ub[i1] = bp_neg<GMODE>(bp_comb<GMODE>(Lch[i1], o1));
                ub[i2] = bp_neg<GMODE>(bp_comb<GMODE>(Lch[i2], o2));
            }
            uint32_t v = 0;
#pragma unroll
            for (int r = 0; r < Q; ++r)
                v |= (bp_neg<GMODE>(su[r]) ? 1u : 0u) << r;
#pragma unroll
            for (int h = 1; h < Q; h <<= 1)
                v ^= (v >> h) & (h == 1 ? 0x55u : (h == 2 ? 0x33u : 0x0Fu));
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const uint32_t pv = __shfl_xor_sync(0xffffffffu, v, s);
                if (!(lane & s))
                    v ^= pv;
            }
            xw[tid] = v;
            __syncthreads();
            uint32_t x = 0;
#pragma unroll
            for (int w2 = 0; w2 < NWARP; ++w2)
                if ((w2 & warp) == warp)
                    x ^= xw[w2 * 32 + lane];
            uint32_t xh = 0;
#pragma unroll
            for (int r = 0; r < Q; ++r)
                xh |= (uint32_t)ub[base + r] << r;
            stop = !__syncthreads_or(x != xh);
        } else if constexpr (RE) {
            // N = 256 (one warp): R[8] = boundary 8 of the R sweep from R[7] (layout C
            // registers, pairs (r, r + 2)) and the channel row; x_hat through the
            // decision bytes into layout A, against the transform of u_hat
            float Lc[Q], R8[Q];
#pragma unroll
            for (int r = 0; r < Q; ++r)
                Lc[r] = Lch[xc(lane, r)];
            stage<GMODE, true, 2>(R7, Lc, R8, lim);
            __syncwarp();
#pragma unroll
            for (int r = 0; r < Q; ++r)
                ub[xc(lane, r)] = bp_neg<GMODE>(bp_comb<GMODE>(Lc[r], R8[r]));
            uint32_t v = 0;
#pragma unroll
            for (int r = 0; r < Q; ++r)
                v |= (bp_neg<GMODE>(su[r]) ? 1u : 0u) << r;
#pragma unroll
            for (int h = 1; h < Q; h <<= 1)
                v ^= (v >> h) & (h == 1 ? 0x55u : (h == 2 ? 0x33u : 0x0Fu));
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const uint32_t pv = __shfl_xor_sync(0xffffffffu, v, s);
                if (!(lane & s))
                    v ^= pv;
            }
            __syncwarp();
            uint32_t xh = 0;
#pragma unroll
            for (int r = 0; r < Q; ++r)
                xh |= (uint32_t)ub[base + r] << r;
            stop = !__any_sync(0xffffffffu, v != xh);
        }
        if (stop || it >= a.i_max)
            break;
    }

    // ---- outputs (as k_bp2) ----
    if (tid == 0) {
        if (a.t_done != nullptr)
            a.t_done[f] = globaltimer();
        a.iters[f] = stop ? it : a.i_max;
        a.conv[f] = stop ? 1 : 0;
    }
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
        // soft_x = L[n] + R[n] (bp.py:164-168); R[n] is formed once here
        if constexpr (LOGN - 1 >= BW) {
            __syncthreads();
            const float *Rp = Rs + (LOGN - 1 - BW) * N;
            for (int p = tid; p < N / 2; p += TPF) {
                const int i1 = p, i2 = p + N / 2;
                float o1, o2;
                bp_pe2<GMODE, true>(Rp[i1], bp_comb<GMODE>(Lch[i2], Rp[i2]), Lch[i1], Rp[i2], lim, o1, o2);
                a.soft_x[(size_t)f * N + i1] = bp_store<GMODE>(bp_comb<GMODE>(Lch[i1], o1));
                a.soft_x[(size_t)f * N + i2] = bp_store<GMODE>(bp_comb<GMODE>(Lch[i2], o2));
            }
        } else {
            // N = 256: R[7] is in layout C registers; boundary 8 pairs registers (r, r + 2)
            float Lc[Q], R8[Q];
#pragma unroll
            for (int r = 0; r < Q; ++r)
                Lc[r] = Lch[wb + xc(lane, r)];
            stage<GMODE, true, 2>(R7, Lc, R8, lim);
#pragma unroll
            for (int r = 0; r < Q; ++r)
                a.soft_x[(size_t)f * N + wb + xc(lane, r)] = bp_store<GMODE>(bp_comb<GMODE>(Lc[r], R8[r]));
        }
    }
    __syncthreads();
    if (a.u_bits != nullptr)
        for (int b = tid; b < 32 * NW; b += TPF) {
            const uint32_t v = __ballot_sync(0xffffffffu, ub[b]);
            if ((b & 31) == 0)
                a.u_bits[(size_t)f * NW + (b >> 5)] = v;
        }
    if (a.payload != nullptr) {
        const int m = a.code.m, MW = (m + 31) >> 5;
        for (int b = tid; b < 32 * MW; b += TPF) {
            const uint32_t v = __ballot_sync(0xffffffffu, b < m && ub[__ldg(a.code.info_pos + b)]);
            if ((b & 31) == 0)
                a.payload[(size_t)f * MW + (b >> 5)] = v;
        }
    }
    if constexpr (!PERS)
        break;
    __syncthreads();
    if (tid == 0) {
        next_f = atomicAdd(a.work, 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    f = next_f;
    }
}

template <int LOGN, int GMODE>
static int launch_bp3_t(const BpArgs &a, cudaStream_t s)
{
    constexpr int TPF = (1 << LOGN) / 8;
    auto kern = k_bp3<LOGN, GMODE, false, false>;
    if (a.stop_mode == 1)
        kern = k_bp3<LOGN, GMODE, true, false>;
    constexpr bool PERS_OK = TPF <= 64;
    // (the re-encode stop runs persistent only at N = 256, one warp per frame)
    const bool pers = PERS_OK && a.work != nullptr && (a.stop_mode != 1 || LOGN == 8);
    if constexpr (PERS_OK)
        if (pers)
            kern = a.stop_mode == 1 ? k_bp3<LOGN, GMODE, true, true> : k_bp3<LOGN, GMODE, false, true>;
    const size_t smem = (size_t)bp3_smem_floats(LOGN) * sizeof(float);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return PC_ERR_CUDA;
    int grid = a.B;
    if (pers) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TPF, smem) != cudaSuccess || per_sm < 1)
            return PC_ERR_CUDA;
        if ((long long)sms * per_sm < grid)
            grid = sms * per_sm;
        if (cudaMemsetAsync(a.work, 0, sizeof(int32_t), s) != cudaSuccess)
            return PC_ERR_CUDA;
    }
    kern<<<grid, TPF, smem, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

// K1 v3 covers N = 256 .. 4096 at 8 nodes per thread (threads_per_frame N/8),
// g_mode 0 (likelihood ratios) and 1 (min-sum), every stop rule.
bool bp3_eligible(const BpArgs &a, int g_mode, int tpf)
{
    const int n = a.code.n;
    if (n < 8 || n > 12 || (g_mode != 0 && g_mode != 1))
        return false;
    if (tpf > 0 && tpf != a.code.N / 8)
        return false;
    return true;
}

int launch_bp3(const BpArgs &a, int g_mode, cudaStream_t s)
{
    if (a.B == 0)
        return PC_OK;
    const int n = a.code.n;
    if (g_mode == 0) {
        switch (n) {
        case 8: return launch_bp3_t<8, 0>(a, s);
        case 9: return launch_bp3_t<9, 0>(a, s);
        case 10: return launch_bp3_t<10, 0>(a, s);
        case 11: return launch_bp3_t<11, 0>(a, s);
        case 12: return launch_bp3_t<12, 0>(a, s);
        }
    } else if (g_mode == 1) {
        switch (n) {
        case 8: return launch_bp3_t<8, 1>(a, s);
        case 9: return launch_bp3_t<9, 1>(a, s);
        case 10: return launch_bp3_t<10, 1>(a, s);
        case 11: return launch_bp3_t<11, 1>(a, s);
        case 12: return launch_bp3_t<12, 1>(a, s);
        }
    }
    return PC_ERR_UNSUPPORTED;
}

} // namespace pc
