// bp2.cu -- K1 v2: BP decoding with register-resident low stages and
// warp-shuffle butterflies (sm_100a).  Same stop cadence as k_bp_decode
// (bp.cu), which restates bp.py:120-217; node update: bp_math.cuh::bp_pe2.
//
// Node ownership: thread t of the frame owns the Q = N / TPF consecutive nodes
// base(t) .. base(t)+Q-1 with base(t) = warp*32Q + lane*Q.  Then
//   * boundaries 1..B (B = log2 Q) join nodes inside one thread: register
//     butterflies, no communication at all;
//   * boundaries B+1..B+5 join nodes of lanes lane ^ 2^(j-1-B) of the same
//     warp: the lane pair splits the PEs (lo lane: nodes 0..Q/2-1, hi lane: the
//     rest), exchanges the operands it lacks with shuffles and evaluates BOTH
//     node updates of its PEs, so the shared operand's exponential is computed
//     once per PE;
//   * only boundaries above BW = B+5 go through shared memory, in radix-4
//     pairs (the nodes b, b+h, b+2h, b+3h are closed under boundaries j and
//     j+1): one CTA barrier per pair.
// The message stages 1..BW-1 of a thread's nodes therefore live in registers
// across iterations (the same thread owns the same nodes in both sweeps), and
// shared memory holds only R[BW..n-1] and L[BW..n] (7 rows, 28 KB at N=1024,
// TPF=256), the R sweep's kept exponentials 2^-|a| for the L sweep (N <= 2048),
// and the decisions.  The frame's channel row arrives by a TMA bulk copy;
// outputs are bit-packed with warp ballots.
#include "args.cuh"
#include "bp_math.cuh"

namespace pc {

template <int V>
struct ilog2 {
    static constexpr int value = 1 + ilog2<V / 2>::value;
};
template <>
struct ilog2<1> {
    static constexpr int value = 0;
};

// Exponential reuse (GMODE 3, the log-domain form): the R sweep's 2^-|a| of every PE at boundaries
// 2..n-1 is kept in shared memory (one float per PE) and reused by the L sweep,
// where a is the PE's second operand: 6 MUFU instead of 7 for those PEs.
__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }
__host__ __device__ constexpr int bp2_base_bytes(int logn, int tpf)
{
    // R rows bw..n-1 and L rows bw..n (bw = log2 Q + 5, i.e. n - bw = log2 TPF - 5), plus N bytes of decisions
    return (2 * (ilog2c(tpf) - 5) + 1) * (1 << logn) * 4 + (1 << logn);
}
// Boundaries 2..n-1 keep their exponentials when all of them (N/2 floats
// each) fit beside the message rows in 225 KB of shared memory.  (Keeping only
// the lower ones at N = 4096 measured 2-4% slower than keeping none:
// tools/bp_tpf_probe.py.)  The KEPT(j) logic supports any prefix count.
__host__ __device__ constexpr int bp2_keep(int logn, int tpf, int gmode)
{
    return gmode == 3 && bp2_base_bytes(logn, tpf) + (logn - 2) * (1 << logn) * 2 <= 225 * 1024 ? logn - 2 : 0;
}
__host__ __device__ constexpr int bp2_keep_bytes(int logn, int tpf, int gmode)
{
    return bp2_keep(logn, tpf, gmode) * (1 << logn) * 2;
}

template <int LOGN, int TPF, int GMODE, bool RE, bool PERS>
__global__ void __launch_bounds__(TPF) k_bp2(const BpArgs a)
{
    constexpr int N = 1 << LOGN;
    constexpr int Q = N / TPF;
    constexpr int B = ilog2<Q>::value;
    constexpr int BW = B + 5;        // last warp-local boundary (TPF >= 32 => BW <= LOGN)
    constexpr int NSR = LOGN - BW;   // shared R rows: stages BW..LOGN-1
    constexpr int NSL = LOGN - BW + 1; // shared L rows: stages BW..LOGN
    constexpr int NREG = BW - 1;     // register stages 1..BW-1
    constexpr int NW = (N + 31) / 32;
    constexpr int NWARP = TPF / 32;
    constexpr int PPT = N / 2 / TPF; // shared-memory boundary elements per thread
    static_assert(TPF >= 32 && Q >= 2 && Q <= 8 && BW <= LOGN, "bp2 geometry");

    extern __shared__ __align__(16) float sm[];
    float *Rs = sm;           // R[BW + r], r < NSR
    float *Ls = sm + NSR * N; // L[BW + r], r < NSL
    uint8_t *ub = reinterpret_cast<uint8_t *>(Ls + NSL * N);
    constexpr int KEEP = bp2_keep(LOGN, TPF, GMODE);
    float *Pa = Ls + NSL * N + N / 4; // kept exponentials, [(j - 2) * Q/2 + k][tid]
    __shared__ uint32_t frz[NW];
    __shared__ uint32_t red[NWARP];
    __shared__ uint32_t xw[RE ? TPF : 1]; // re-encode stop: the warp-transformed bits of each thread

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int f = blockIdx.x;
    const BpLim lim = bp_lim<GMODE>(a.llr_max); // clip bounds in the mode's message domain (bp_math.cuh)
    const int base = warp * 32 * Q + lane * Q;

    // the frame's channel LLRs land in L[n] by a TMA bulk copy while the
    // threads clear the message rows; then each thread scales and clips its part
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
    // PERS: the CTA loops over frames taken from a work counter (frames have
    // 1..i_max iterations; the counter keeps every CTA slot busy)
    while (f < a.B) {
    if (tid == 0)
        tma_load_1d(Lch, a.llr + (size_t)f * N, N * sizeof(float), &ch_bar);
    // (the R rows are written by the R sweep before any read; only L starts at 0)
    for (int i = tid; i < (NSL - 1) * N; i += TPF)
        Ls[i] = bp_zero<GMODE>();
    mbar_wait(&ch_bar, phase);
    phase ^= 1u;
    for (int i = 4 * tid; i < N; i += 4 * TPF) {
        const float4 v = *reinterpret_cast<const float4 *>(Lch + i);
        *reinterpret_cast<float4 *>(Lch + i) = make_float4(bp_load<GMODE>(v.x, a.llr_max), bp_load<GMODE>(v.y, a.llr_max),
                                                          bp_load<GMODE>(v.z, a.llr_max), bp_load<GMODE>(v.w, a.llr_max));
    }
    float Rr[NREG][Q], Lr[NREG][Q];
#pragma unroll
    for (int s = 0; s < NREG; ++s)
#pragma unroll
        for (int r = 0; r < Q; ++r)
            Rr[s][r] = Lr[s][r] = bp_zero<GMODE>();
    uint32_t col[Q];
#pragma unroll
    for (int r = 0; r < Q; ++r)
        col[r] = a.stop_mode == 0 ? __ldg(a.code.crc_cols + base + r) : 0u;
    __syncthreads();
    const uint32_t fw = frz[base >> 5] >> (base & 31);
    float pri[Q];
#pragma unroll
    for (int r = 0; r < Q; ++r)
        pri[r] = ((fw >> r) & 1u) ? bp_prior<GMODE>(lim) : bp_zero<GMODE>();

    // compile-time stage accessors (every loop below is fully unrolled, so the
    // register arrays are indexed with constants)
#define KEPT(j) ((j) >= 2 && (j) - 2 < KEEP)
#define PA(j, k) Pa[(((j) - 2) * (Q / 2) + (k)) * TPF + tid]
#define PAP(j, p) Pa[((j) - 2) * (N / 2) + (p)] // shared-memory boundaries: indexed by PE
    const float pprior = GMODE == 3 ? ex2_approx(-lim.hi) : 0.0f; // 2^-|R[0]| of a frozen node
#define RGET(s, r) ((s) == 0 ? pri[r] : ((s) <= NREG ? Rr[(s) > 0 ? (s) - 1 : 0][r] : Rs[((s) - BW) * N + base + (r)]))
#define LGET(s, r) ((s) <= NREG ? Lr[(s) > 0 ? (s) - 1 : 0][r] : Ls[((s) - BW) * N + base + (r)])

    float su[Q];
    int it = 0;
    bool stop = false;
    for (;;) {
        ++it;
        // ================= R sweep =================
#pragma unroll
        for (int j = 1; j <= B; ++j) { // inside the thread
            const int h = 1 << (j - 1);
#pragma unroll
            for (int r1 = 0; r1 < Q; ++r1) {
                if (r1 & h)
                    continue;
                const int r2 = r1 + h;
                const float av = RGET(j - 1, r1), r2v = RGET(j - 1, r2), l1 = LGET(j, r1), l2 = LGET(j, r2);
                if (KEPT(j)) {
                    float px;
                    bp_pe2_keep(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, Rr[j - 1][r1], Rr[j - 1][r2], px);
                    PA(j, ((r1 >> j) << (j - 1)) | (r1 & (h - 1))) = px;
                } else {
                    bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, Rr[j - 1][r1], Rr[j - 1][r2]);
                }
            }
        }
#pragma unroll
        for (int j = B + 1; j <= BW; ++j) { // across lanes of the warp
            if (j == LOGN)
                break; // R[n] is not read by the sweeps
            const int msk = 1 << (j - 1 - B);
            const bool hi = lane & msk;
            // Lane pair (lo = node i1, hi = node i2): the lo lane computes both outputs
            // of nodes 0..Q/2-1, the hi lane those of nodes Q/2..Q-1, so the shared
            // operand's exponential is evaluated once per PE (bp_pe2).
            float Rn[Q];
#pragma unroll
            for (int k = 0; k < Q / 2; ++k) {
                const float Rk = RGET(j - 1, k), Rh = RGET(j - 1, k + Q / 2);
                const float Lk = LGET(j, k), Lh = LGET(j, k + Q / 2);
                // send the partner the node it owns, keep mine (k on the lo lane, k + Q/2 on hi)
                const float pr = __shfl_xor_sync(0xffffffffu, hi ? Rk : Rh, msk);
                const float pl = __shfl_xor_sync(0xffffffffu, hi ? Lk : Lh, msk);
                const float myR = hi ? Rh : Rk, myL = hi ? Lh : Lk;
                // (a, r2, l1, l2) of the PE at my node
                const float av = hi ? pr : myR, r2v = hi ? myR : pr, l1 = hi ? pl : myL, l2 = hi ? myL : pl;
                float o1, o2;
                if (KEPT(j)) {
                    float px;
                    bp_pe2_keep(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, o1, o2, px);
                    PA(j, k) = px;
                } else {
                    bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, o1, o2);
                }
                const float back = __shfl_xor_sync(0xffffffffu, hi ? o1 : o2, msk); // my output the partner computed
                Rn[k] = hi ? back : o1;
                Rn[k + Q / 2] = hi ? o2 : back;
            }
#pragma unroll
            for (int r = 0; r < Q; ++r) {
                if (j <= NREG)
                    Rr[j - 1][r] = Rn[r];
                else
                    Rs[(j - BW) * N + base + r] = Rn[r];
            }
        }
        __syncthreads();
        // Shared-memory boundaries in pairs (j, j+1): the four nodes b, b+h, b+2h,
        // b+3h (h = 2^(j-1)) are closed under both boundaries, so one thread
        // runs both PEs of j and then both of j+1 with one barrier per pair.
#pragma unroll
        for (int j = BW + 1; j <= LOGN - 1; j += (Q >= 4 ? 2 : 1)) {
            const int h = 1 << (j - 1);
            const float *Rp = Rs + (j - 1 - BW) * N;
            float *Rd = Rs + (j - BW) * N;
            const float *Lj = Ls + (j - BW) * N;
            if (Q >= 4 && j + 1 <= LOGN - 1) { // (Q >= 4: a 4-node group per thread)
                float *Rd2 = Rs + (j + 1 - BW) * N;
                const float *Lj2 = Ls + (j + 1 - BW) * N;
#pragma unroll
                for (int q = 0; q < Q / 4; ++q) {
                    const int g = tid + q * TPF;
                    const int n0 = ((g >> (j - 1)) << (j + 1)) | (g & (h - 1));
                    const int n1 = n0 + h, n2 = n0 + 2 * h, n3 = n0 + 3 * h;
                    float o[4];
#pragma unroll
                    for (int e = 0; e < 2; ++e) { // boundary j: (n0, n1), (n2, n3)
                        const int i1 = e ? n2 : n0, i2 = i1 + h;
                        const float av = Rp[i1], r2v = Rp[i2], l1 = Lj[i1], l2 = Lj[i2];
                        if (KEPT(j)) {
                            float px;
                            bp_pe2_keep(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, o[2 * e], o[2 * e + 1], px);
                            PAP(j, ((i1 >> j) << (j - 1)) | (i1 & (h - 1))) = px;
                        } else {
                            bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, o[2 * e], o[2 * e + 1]);
                        }
                    }
                    Rd[n0] = o[0];
                    Rd[n1] = o[1];
                    Rd[n2] = o[2];
                    Rd[n3] = o[3];
#pragma unroll
                    for (int e = 0; e < 2; ++e) { // boundary j + 1: (n0, n2), (n1, n3)
                        const int i1 = e ? n1 : n0, i2 = i1 + 2 * h;
                        const float av = o[e], r2v = o[e + 2], l1 = Lj2[i1], l2 = Lj2[i2];
                        float p1, p2;
                        if (KEPT(j + 1)) {
                            float px;
                            bp_pe2_keep(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, p1, p2, px);
                            PAP(j + 1, ((i1 >> (j + 1)) << j) | (i1 & (2 * h - 1))) = px;
                        } else {
                            bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, p1, p2);
                        }
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
                    if (KEPT(j)) {
                        float px;
                        bp_pe2_keep(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, o1, o2, px);
                        PAP(j, p) = px;
                    } else {
                        bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, o1, o2);
                    }
                    Rd[i1] = o1;
                    Rd[i2] = o2;
                }
            }
            __syncthreads();
        }
        // ================= L sweep =================
        // shared-memory boundaries top-down in pairs (j + 1, j), as in the R sweep
#pragma unroll
        for (int jt = LOGN; jt >= BW + 1; jt -= (Q >= 4 ? 2 : 1)) {
            if (Q >= 4 && jt - 1 >= BW + 1) {
                const int j = jt - 1;
                const int h = 1 << (j - 1);
                const float *Rj = Rs + (j - BW) * N;      // R[j]   (a, r2 of boundary j + 1)
                const float *Rp = Rs + (j - 1 - BW) * N;  // R[j-1] (a, r2 of boundary j)
                const float *Lt = Ls + (j + 1 - BW) * N;  // L[j+1]
                float *Lm = Ls + (j - BW) * N;            // L[j]
                float *Ld = Ls + (j - 1 - BW) * N;        // L[j-1]
#pragma unroll
                for (int q = 0; q < Q / 4; ++q) {
                    const int g = tid + q * TPF;
                    const int n0 = ((g >> (j - 1)) << (j + 1)) | (g & (h - 1));
                    const int n1 = n0 + h, n2 = n0 + 2 * h, n3 = n0 + 3 * h;
                    float m[4]; // L[j] at n0..n3
#pragma unroll
                    for (int e = 0; e < 2; ++e) { // boundary j + 1: (n0, n2), (n1, n3)
                        const int i1 = e ? n1 : n0, i2 = i1 + 2 * h;
                        const float av = Rj[i1], r2v = Rj[i2], l1 = Lt[i1], l2 = Lt[i2];
                        float o1, o2;
                        if (KEPT(j + 1))
                            bp_pe2_p2(l1, bp_comb<GMODE>(l2, r2v), av, PAP(j + 1, ((i1 >> (j + 1)) << j) | (i1 & (2 * h - 1))), l2,
                                      lim, o1, o2);
                        else
                            bp_pe2<GMODE, false, KEEP == 0 && GMODE == 3>(l1, bp_comb<GMODE>(l2, r2v), av, l2, lim, o1, o2);
                        m[e] = o1;
                        m[e + 2] = o2;
                    }
                    Lm[n0] = m[0];
                    Lm[n1] = m[1];
                    Lm[n2] = m[2];
                    Lm[n3] = m[3];
#pragma unroll
                    for (int e = 0; e < 2; ++e) { // boundary j: (n0, n1), (n2, n3)
                        const int i1 = e ? n2 : n0, i2 = i1 + h;
                        const float av = Rp[i1], r2v = Rp[i2], l1 = m[2 * e], l2 = m[2 * e + 1];
                        float o1, o2;
                        if (KEPT(j))
                            bp_pe2_p2(l1, bp_comb<GMODE>(l2, r2v), av, PAP(j, ((i1 >> j) << (j - 1)) | (i1 & (h - 1))), l2, lim, o1,
                                      o2);
                        else
                            bp_pe2<GMODE, false, KEEP == 0 && GMODE == 3>(l1, bp_comb<GMODE>(l2, r2v), av, l2, lim, o1, o2);
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
                    if (KEPT(j))
                        bp_pe2_p2(l1, bp_comb<GMODE>(l2, r2v), av, PAP(j, p), l2, lim, o1, o2);
                    else
                        bp_pe2<GMODE, false, KEEP == 0 && GMODE == 3>(l1, bp_comb<GMODE>(l2, r2v), av, l2, lim, o1, o2);
                    Ld[i1] = o1;
                    Ld[i2] = o2;
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int j = BW; j >= B + 1; --j) {
            const int msk = 1 << (j - 1 - B);
            const bool hi = lane & msk;
            float Ln[Q];
#pragma unroll
            for (int k = 0; k < Q / 2; ++k) {
                const float Rk = RGET(j - 1, k), Rh = RGET(j - 1, k + Q / 2);
                const float Lk = LGET(j, k), Lh = LGET(j, k + Q / 2);
                // send the partner the node it owns, keep mine (k on the lo lane, k + Q/2 on hi)
                const float pr = __shfl_xor_sync(0xffffffffu, hi ? Rk : Rh, msk);
                const float pl = __shfl_xor_sync(0xffffffffu, hi ? Lk : Lh, msk);
                const float myR = hi ? Rh : Rk, myL = hi ? Lh : Lk;
                // (a, r2, l1, l2) of the PE at my node
                const float av = hi ? pr : myR, r2v = hi ? myR : pr, l1 = hi ? pl : myL, l2 = hi ? myL : pl;
                float o1, o2;
                if (KEPT(j))
                    bp_pe2_p2(l1, bp_comb<GMODE>(l2, r2v), av, PA(j, k), l2, lim, o1, o2);
                else
                    bp_pe2<GMODE, false, KEEP == 0 && GMODE == 3>(l1, bp_comb<GMODE>(l2, r2v), av, l2, lim, o1, o2);
                const float back = __shfl_xor_sync(0xffffffffu, hi ? o1 : o2, msk); // my output the partner computed
                Ln[k] = hi ? back : o1;
                Ln[k + Q / 2] = hi ? o2 : back;
            }
#pragma unroll
            for (int r = 0; r < Q; ++r)
                Lr[j - 2][r] = Ln[r]; // j - 1 >= B >= 1 is a register stage
        }
#pragma unroll
        for (int j = B; j >= 1; --j) {
            const int h = 1 << (j - 1);
#pragma unroll
            for (int r1 = 0; r1 < Q; ++r1) {
                if (r1 & h)
                    continue;
                const int r2 = r1 + h;
                const float av = RGET(j - 1, r1), r2v = RGET(j - 1, r2), l1 = LGET(j, r1), l2 = LGET(j, r2);
                float o1, o2;
                if (KEPT(j))
                    bp_pe2_p2(l1, bp_comb<GMODE>(l2, r2v), av, PA(j, ((r1 >> j) << (j - 1)) | (r1 & (h - 1))), l2, lim, o1, o2);
                else if (GMODE == 3 && j == 1)
                    bp_pe2_p2(l1, bp_comb<GMODE>(l2, r2v), av, av != 0.0f ? pprior : 1.0f, l2, lim, o1, o2); // R[0] prior
                else
                    bp_pe2<GMODE, false, KEEP == 0 && GMODE == 3>(l1, bp_comb<GMODE>(l2, r2v), av, l2, lim, o1, o2);
                if (j > 1) {
                    Lr[j - 2][r1] = o1;
                    Lr[j - 2][r2] = o2;
                } else {
                    su[r1] = bp_comb<GMODE>(o1, av); // soft_u = L[0] + R[0]
                    su[r2] = bp_comb<GMODE>(o2, r2v);
                }
            }
        }
        // ================= stop rule (crc or none) =================
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
            {
                // re-encode stop (bp.py:187): polar_transform(hard(soft_u)) == hard(L[n] + R[n]).
                // R[n] comes from this iteration's R[n-1] row (the L sweep leaves it
                // alone); x_hat lands as bytes in ub.  The transform of the thread's
                // Q bits runs in registers (in-thread, then lane shuffles); the
                // cross-warp stages read the other warps' words once: x_w = XOR of
                // v_w' over the warps w' whose index contains w's bits.
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
            }
        }
        if (stop || it >= a.i_max)
            break;
    }

    // ---- outputs ----
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
    if constexpr (LOGN - 1 >= BW) {
        // soft_x = L[n] + R[n] (bp.py:164-168); R[n] is not needed by the sweeps,
        // so it is formed once here from the final R[n-1] row (shared memory).
        if (a.soft_x != nullptr) {
            __syncthreads();
            const float *Rp = Rs + (LOGN - 1 - BW) * N;
            for (int p = tid; p < N / 2; p += TPF) {
                const int i1 = p, i2 = p + N / 2;
                float o1, o2;
                bp_pe2<GMODE, true>(Rp[i1], bp_comb<GMODE>(Lch[i2], Rp[i2]), Lch[i1], Rp[i2], lim, o1, o2);
                a.soft_x[(size_t)f * N + i1] = bp_store<GMODE>(bp_comb<GMODE>(Lch[i1], o1));
                a.soft_x[(size_t)f * N + i2] = bp_store<GMODE>(bp_comb<GMODE>(Lch[i2], o2));
            }
        }
    } else {
        // BW = n (one warp per frame at N = 128): R[n-1] is a register stage, so
        // R[n] comes from the same lane-pair exchange as the R sweep's boundary n
        if (a.soft_x != nullptr) {
            constexpr int j = LOGN;
            const int msk = 1 << (j - 1 - B);
            const bool hi = lane & msk;
#pragma unroll
            for (int k = 0; k < Q / 2; ++k) {
                const float Rk = RGET(j - 1, k), Rh = RGET(j - 1, k + Q / 2);
                const float Lk = LGET(j, k), Lh = LGET(j, k + Q / 2);
                const float pr = __shfl_xor_sync(0xffffffffu, hi ? Rk : Rh, msk);
                const float pl = __shfl_xor_sync(0xffffffffu, hi ? Lk : Lh, msk);
                const float myR = hi ? Rh : Rk, myL = hi ? Lh : Lk;
                const float av = hi ? pr : myR, r2v = hi ? myR : pr, l1 = hi ? pl : myL, l2 = hi ? myL : pl;
                float o1, o2;
                bp_pe2<GMODE, true>(av, bp_comb<GMODE>(l2, r2v), l1, r2v, lim, o1, o2);
                const float back = __shfl_xor_sync(0xffffffffu, hi ? o1 : o2, msk);
                const float rk = hi ? back : o1, rh = hi ? o2 : back; // R[n] at my nodes k, k + Q/2
                a.soft_x[(size_t)f * N + base + k] = bp_store<GMODE>(bp_comb<GMODE>(Lk, rk));
                a.soft_x[(size_t)f * N + base + k + Q / 2] = bp_store<GMODE>(bp_comb<GMODE>(Lh, rh));
            }
        }
    }
    __syncthreads();
    // bit-pack with warp ballots: thread b of the pass owns bit b (coalesced
    // info_pos reads, one store per 32 bits)
    if (a.u_bits != nullptr)
        for (int b = tid; b < 32 * NW; b += TPF) {
            const uint32_t v = __ballot_sync(0xffffffffu, b < N && ub[b]);
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
    __syncthreads(); // this frame's shared memory is dead
    if (tid == 0) {
        next_f = atomicAdd(a.work, 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // generic writes before the next TMA
    }
    __syncthreads();
    f = next_f;
    }
}

#undef RGET
#undef LGET
#undef PA
#undef PAP
#undef KEPT

// Default threads per frame (measured, tools/bp_gmode_probe.py and
// tools/bp_tpf_probe.py).  The likelihood-ratio form (g_mode 0) is fastest at
// Q = 8 nodes per thread at every N (N=1024: 3265 / 3058 / 2568 Gg/s at 128 /
// 256 / 512 threads); the re-encode stop needs R[n-1] in shared memory, i.e.
// at least 64 threads.  The log-domain forms keep the round-1 settings.
static int bp2_default_tpf(int N, int gmode, int stop_mode)
{
    if (gmode == 0) {
        const int t = N / 8 > 32 ? N / 8 : 32;
        return stop_mode == 1 && t < 64 ? 64 : t;
    }
    return N >= 4096 ? 512 : (N / 4 >= 256 ? 256 : N / 4);
}

static size_t bp2_smem_bytes(int logn, int tpf)
{
    const int N = 1 << logn;
    int q = N / tpf, b = 0;
    while ((1 << b) < q)
        ++b;
    const int bw = b + 5;
    return (size_t)((logn - bw) + (logn - bw + 1)) * N * sizeof(float) + N;
}

template <int LOGN, int TPF, int GMODE>
static int launch_bp2_t(const BpArgs &a, cudaStream_t s)
{
    // the re-encode stop is its own instantiation (its registers would cost the
    // CRC kernel an occupancy step at N = 1024)
    auto kern = k_bp2<LOGN, TPF, GMODE, false, false>;
    if constexpr (GMODE != 2 && TPF >= 64)
        if (a.stop_mode == 1)
            kern = k_bp2<LOGN, TPF, GMODE, true, false>;
    // Persistent CTAs where a CTA is one or two warps (N <= 512 at the default
    // thread counts): there, frames of 1..i_max iterations leave CTA slots
    // empty between frames (measured: 27% -> 44% warps active at N = 128,
    // 14% faster); with 8+ warps per CTA the two forms time the same.
    constexpr bool PERS_OK = GMODE != 2 && TPF <= 64;
    const bool pers = PERS_OK && a.work != nullptr && a.stop_mode != 1;
    if constexpr (PERS_OK)
        if (pers)
            kern = k_bp2<LOGN, TPF, GMODE, false, true>;
    const size_t smem = bp2_smem_bytes(LOGN, TPF) + bp2_keep_bytes(LOGN, TPF, GMODE);
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

template <int LOGN, int GMODE>
static int launch_bp2_n(const BpArgs &a, int tpf, cudaStream_t s)
{
    constexpr int N = 1 << LOGN;
    constexpr int LO = N / 8 > 32 ? N / 8 : 32; // Q <= 8 nodes per thread (Q = 16 needs ~120+ registers)
    constexpr int HI = N / 2;                   // Q >= 2
    if (tpf <= 0)
        tpf = bp2_default_tpf(N, GMODE, a.stop_mode);
    if (tpf < LO || tpf > HI)
        return PC_ERR_UNSUPPORTED;
#define PC_BP2_CASE(T)                                                                                                 \
    case T: return launch_bp2_t<LOGN, (T < LO ? LO : (T > HI ? HI : T)), GMODE>(a, s);
    switch (tpf) {
        PC_BP2_CASE(32)
        PC_BP2_CASE(64)
        PC_BP2_CASE(128)
        PC_BP2_CASE(256)
        PC_BP2_CASE(512)
        PC_BP2_CASE(1024)
    default: return PC_ERR_UNSUPPORTED;
    }
#undef PC_BP2_CASE
}

// K1 v2 covers N = 128 .. 4096 with every stop rule (re-encode: TPF >= 64) and
// both soft outputs; the shared-memory kernel in bp.cu serves N < 128, the
// re-encode stop at TPF = 32 and the kernel = 1 knob.
// N = 4096 runs one 512-thread CTA per frame (Q = 8): 9 shared rows (144 KB),
// no kept exponentials, one CTA per SM.
bool bp2_eligible(const BpArgs &a, int g_mode, int tpf)
{
    const int N = a.code.N;
    const int lo = N / 8 > 32 ? N / 8 : 32;
    // soft outputs at every N: bp_decode (per frame, soft_u and soft_x) and
    // bp_decode_batch / the hybrid run the same kernel, so they decide alike
    if (!(a.code.n >= 7 && a.code.n <= 12 && (tpf <= 0 || (tpf >= lo && tpf <= N / 2))))
        return false;
    if (a.stop_mode != 1)
        return true;
    // the re-encode stop needs R[n-1] in shared memory: log2 TPF >= 6
    const int t = tpf > 0 ? tpf : bp2_default_tpf(N, g_mode, a.stop_mode);
    return t >= 64;
}

int launch_bp2(const BpArgs &a, int g_mode, int tpf, cudaStream_t s)
{
    if (a.B == 0)
        return PC_OK;
    if (!bp2_eligible(a, g_mode, tpf) || (g_mode == 2 && a.stop_mode == 1))
        return PC_ERR_UNSUPPORTED;
    const int n = a.code.n;
    if (g_mode == 2) { // exact g, per-g form (parity studies)
        switch (n) {
        case 10: return launch_bp2_n<10, 2>(a, tpf, s);
        case 11: return launch_bp2_n<11, 2>(a, tpf, s);
        }
        return PC_ERR_UNSUPPORTED;
    }
    if (g_mode == 3) { // the round-1 log-domain form (A/B knob)
        switch (n) {
        case 7: return launch_bp2_n<7, 3>(a, tpf, s);
        case 8: return launch_bp2_n<8, 3>(a, tpf, s);
        case 9: return launch_bp2_n<9, 3>(a, tpf, s);
        case 10: return launch_bp2_n<10, 3>(a, tpf, s);
        case 11: return launch_bp2_n<11, 3>(a, tpf, s);
        case 12: return launch_bp2_n<12, 3>(a, tpf, s);
        }
        return PC_ERR_UNSUPPORTED;
    }
    if (g_mode == 0) {
        switch (n) {
        case 7: return launch_bp2_n<7, 0>(a, tpf, s);
        case 8: return launch_bp2_n<8, 0>(a, tpf, s);
        case 9: return launch_bp2_n<9, 0>(a, tpf, s);
        case 10: return launch_bp2_n<10, 0>(a, tpf, s);
        case 11: return launch_bp2_n<11, 0>(a, tpf, s);
        case 12: return launch_bp2_n<12, 0>(a, tpf, s);
        }
    } else {
        switch (n) {
        case 7: return launch_bp2_n<7, 1>(a, tpf, s);
        case 8: return launch_bp2_n<8, 1>(a, tpf, s);
        case 9: return launch_bp2_n<9, 1>(a, tpf, s);
        case 10: return launch_bp2_n<10, 1>(a, tpf, s);
        case 11: return launch_bp2_n<11, 1>(a, tpf, s);
        case 12: return launch_bp2_n<12, 1>(a, tpf, s);
        }
    }
    return PC_ERR_UNSUPPORTED;
}

} // namespace pc
