// scl3.cuh -- K3 v3: CRC-aided SCL with register-resident leaf blocks (sm_100a).
//
// Same decoder as scl.cu (reference _kernels.py:144-333 + scl.py:177-191, with
// the reference's logical slot numbering and (metric, candidate index) order),
// restructured around blocks of 2^T = 32 leaves (T = PC_SCL3_T, scl3_decl.cuh):
//
//   * upper descent, once per block: tree levels >= T+1 live in shared memory
//     with lazy slot pointers (as in v2) and produce the block's level-T LLRs
//     straight into registers;
//   * the leaves of a block run on registers only: levels 0..T-1, the partial
//     sums of those levels (one word) and the per-leaf control.  One copy of
//     the leaf code serves every leaf (runtime leaf index, warp-uniform
//     branches) -- an unrolled block overflows the instruction cache.  A clone
//     copies the parent's still-readable register levels with shuffles (the
//     reference's eager copy, _kernels.py:288-303);
//   * survivor selection at a full list (P == L): every agreeing child below
//     the best disagreeing one is kept and every disagreeing child above the
//     worst agreeing one dropped (two warp reductions, redux.sync at L = 32);
//     the remaining slots go to the smallest of the uncertain set, ranked in
//     shared memory.  The result is exactly the L smallest (metric, index)
//     pairs (_kernels.py:253-267);
//   * the frozen prefix (one path, all decisions 0) is decoded element-parallel
//     by the whole warp (frozen_prefix) with bit-identical state;
//   * the CRC syndrome of every path is carried incrementally (one XOR of the
//     position's syndrome column per decided 1) and copied on clone, so the
//     CRC-aided winner rule (scl.py:181-191) needs no stored decisions;
//   * decisions are stored as 32-bit windows with an ancestor lane per window
//     (a traceback in the caller's workspace); only the winner's path is
//     reconstructed at the end.
#pragma once
#include "args.cuh"
#include "scl_math.cuh"
#include "scl3_decl.cuh"

namespace pc {

#ifdef SCL3_STATS
// development counters (tools/scl3_stats.py): full-list selections, those with an
// uncertain set, those settled by one swap, those ranked, clones
static __device__ unsigned long long g_scl3_stats[8];
#define S3_COUNT(i) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_scl3_stats[i], 1ull); } while (0)
#else
#define S3_COUNT(i) do { } while (0)
#endif

namespace s3 {


__device__ __forceinline__ int sl32(uint32_t p, int s) { return (int)((p >> (5 * (s - T - 1))) & 31u); }
__device__ __forceinline__ uint32_t set32(uint32_t p, int s, int v)
{
    const int sh = 5 * (s - T - 1);
    return (p & ~(31u << sh)) | ((uint32_t)v << sh);
}
__device__ __forceinline__ int sl64(uint64_t p, int s) { return (int)((p >> (5 * (s - T))) & 31u); }
__device__ __forceinline__ uint64_t set64(uint64_t p, int s, int v)
{
    const int sh = 5 * (s - T);
    return (p & ~(31ull << sh)) | ((uint64_t)v << sh);
}

// compile-time trailing zeros / ones of a small non-negative integer
__host__ __device__ constexpr int ctz_c(int v) { return (v & 1) ? 0 : 1 + ctz_c(v >> 1); }
__host__ __device__ constexpr int cto_c(int v) { return (v & 1) ? 1 + cto_c(v >> 1) : 0; }

// Order-preserving key of a non-negative fp32 metric (metrics only grow from 0).
__device__ __forceinline__ uint32_t mkey(float m) { return __float_as_uint(m); }

template <int L>
__device__ __forceinline__ uint32_t gmax_u(uint32_t v)
{
    if constexpr (L == 32) {
        return __reduce_max_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int off = 1; off < L; off <<= 1)
            v = max(v, (uint32_t)__shfl_xor_sync(0xffffffffu, v, off));
        return v;
    }
}

template <int L>
__device__ __forceinline__ uint32_t gmin_u(uint32_t v)
{
    if constexpr (L == 32) {
        return __reduce_min_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int off = 1; off < L; off <<= 1)
            v = min(v, (uint32_t)__shfl_xor_sync(0xffffffffu, v, off));
        return v;
    }
}

template <int L>
__device__ __forceinline__ int gmax_i(int v)
{
    if constexpr (L == 32) {
        return __reduce_max_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int off = 1; off < L; off <<= 1)
            v = max(v, __shfl_xor_sync(0xffffffffu, v, off));
        return v;
    }
}

template <int L>
__device__ __forceinline__ int gmin_i(int v)
{
    if constexpr (L == 32) {
        return __reduce_min_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int off = 1; off < L; off <<= 1)
            v = min(v, __shfl_xor_sync(0xffffffffu, v, off));
        return v;
    }
}

template <int L>
__device__ __forceinline__ int gsum_i(int v)
{
    if constexpr (L == 32) {
        return __reduce_add_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int off = 1; off < L; off <<= 1)
            v += __shfl_xor_sync(0xffffffffu, v, off);
        return v;
    }
}

// Frozen prefix (leaves [0, E), one path alive): every decision is 0, so every
// node value depends on the channel only and the tree is walked breadth-first,
// element-parallel over the warp, in the slots of lanes 1..31 (unused while one
// path is alive).  Same f / g(u = 0) arithmetic as the block walk; the last node
// of each stored level goes to lane 0's slot, lane 0's partial sums are zeroed
// (the codeword of an all-frozen prefix is 0), and the returned metric is the
// same sequential sum of the u = 0 increments: the state is bit-identical to
// walking the E / 2^T blocks.
template <bool FEX>
__device__ __noinline__ float frozen_prefix(const float *ch, float *llr, uint32_t *ps, int n, int tp, int ss, int psw,
                                            int E, int metric_exact, int lane)
{
    const int N = 1 << n;
    float *sA = llr + ss, *sB = sA + N;
    const float *Pv = ch;
    float *out = sA;
    for (int s = n - 1; s >= 0; --s) {
        const int w = 1 << s;
        const int tot = ((E + w - 1) >> s) << s;
        for (int idx = lane; idx < tot; idx += 32) {
            const int k = idx >> s, t = idx & (w - 1);
            const float *pp = Pv + ((k >> 1) << (s + 1));
            const float A = pp[t], Bv = pp[t + w];
            out[idx] = (k & 1) ? Bv + A : scl_f<FEX>(A, Bv);
        }
        __syncwarp();
        if (s >= T + 1 && s <= tp) {
            const int kk = (E - 1) >> s;
            for (int t = lane; t < w; t += 32)
                llr[llo(s) + t] = out[(kk << s) + t];
        }
        Pv = out;
        out = (out == sA) ? sB : sA;
        __syncwarp();
    }
    for (int i = lane; i < E; i += 32) {
        float i0v, i1v;
        metric_incs(Pv[i], metric_exact, i0v, i1v);
        out[i] = i0v;
    }
    for (int q = lane; q < psw; q += 32)
        ps[q] = 0u;
    __syncwarp();
    float m = 0.0f;
    if (lane == 0)
        for (int i = 0; i < E; ++i)
            m += out[i];
    __syncwarp();
    return m;
}

} // namespace s3

#ifndef SCL3_CN
#define SCL3_CN 1
#endif
#ifndef SCL3_CN_ME
#define SCL3_CN_ME 1
#endif
#ifndef PC_SCL3_MAXREG
#define PC_SCL3_MAXREG 0
#endif
#if PC_SCL3_MAXREG > 0
#define PC_SCL3_BOUNDS __maxnreg__(PC_SCL3_MAXREG)
#else
#define PC_SCL3_BOUNDS __launch_bounds__(128)
#endif

// CN > 0: the code length 2^CN and the slot layout that scl3_prepare derives
// from it are compile-time constants (the launcher checks them), so the
// address arithmetic folds into immediates.
template <int CN, int NV>
struct Scl3Geom {
    static constexpr int tp = CN - 1 - NV;
    static constexpr int lw = tp >= s3::T + 1 ? (1 << (tp + 1)) - (1 << (s3::T + 1)) : 0;
    static constexpr int ss = ((lw + 7) & ~7) + 4;
    static constexpr int psw = ((5 - s3::T) + (1 << (CN - 5)) - 1) | 1;
};

template <int L, bool FEX, int NV, int CN = 0>
__global__ void PC_SCL3_BOUNDS k_scl3(const SclArgs a)
{
    using namespace s3;
    constexpr int F = 32 / L;
    constexpr uint32_t FULL = 0xffffffffu;
    extern __shared__ __align__(16) uint32_t smw[];
    using G = Scl3Geom<CN ? CN : 10, NV>;
    const int n = CN ? CN : a.code.n;
    const int N = CN ? (1 << CN) : a.code.N;
    const int tp = CN ? G::tp : a.tp, ss = CN ? G::ss : a.ss, psw = CN ? G::psw : a.psw, W = a.uhs;
    const int lane = threadIdx.x & 31;
    uint32_t *wb = smw + (size_t)(threadIdx.x >> 5) * a.warp_words;
    float *llr = reinterpret_cast<float *>(wb);
    uint32_t *ps = wb + a.o_ps;
    // decision traceback of this warp in the workspace: W x 32 words + W x 32 ancestor bytes
    uint32_t *tb = a.tbg + (size_t)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (size_t)W * 40;
    uint8_t *tba = reinterpret_cast<uint8_t *>(tb + W * 32);
    float *cand = reinterpret_cast<float *>(wb + a.o_cand);
    uint32_t *wrow = wb + a.o_wrow;
    float *chs = reinterpret_cast<float *>(wb + a.o_ch);
    constexpr bool CK = CN && SCL3_CN_ME; // the compiled-in defaults (see scl3_geom_is)
    const bool ch_smem = CK ? false : a.o_ch >= 0;

    const int grp = lane / L, gbase = grp * L, pl = lane - gbase;
    // the list size: L (the lanes per frame) or, for a list size that is not a
    // power of two, fewer (lanes Lc..L-1 of a frame group never hold a path)
    const int Lc = CK ? L : (a.list_cap > 0 && a.list_cap < L ? a.list_cap : L);
    const uint32_t gmask_lo = (L == 32) ? FULL : ((1u << L) - 1u);
    const int total = a.count != nullptr ? *a.count : a.B;
    float *own = llr + lane * ss;
    uint32_t *pown = ps + lane * psw;
    float *cg = cand + grp * 4 * L;
    const uint32_t *frzg = a.code.frozen_bits;
    // (the compiled-in geometries also fix the default knobs: CRC on, no
    // decision-aided positions, exact metric)
    const uint32_t *damg = CK ? nullptr : a.code.da_bits;
    const uint32_t *colg = a.code.crc_cols;
    const bool use_crc = CK ? true : a.code.crc_width > 0;

    // blocks before the first non-frozen position: decoded element-parallel (below)
    // (from the code struct, not a device load: a load here costs the block walk
    // ~20% through its code generation)
    const int nb0 = (L == 32 && (CK || a.prefix)) ? a.code.first_info >> T : 0;

    uint32_t lp32 = 0;
    uint64_t lp64 = 0;
    for (int f = 0; f < 6; ++f)
        lp32 |= (uint32_t)lane << (5 * f);
    for (int f = 0; f < 12; ++f)
        lp64 |= (uint64_t)lane << (5 * f);

    for (;;) {
        int base = 0;
        if (lane == 0)
            base = atomicAdd(a.work, F);
        base = __shfl_sync(FULL, base, 0);
        if (base >= total)
            break;
        const int qi = base + grp;
        const bool grp_live = qi < total;
        const int frame = grp_live ? (a.queue != nullptr ? a.queue[qi] : qi) : 0;
        const float *ch;
        if (ch_smem) {
            float *mine = chs + grp * N;
            const float *g = a.llr + (size_t)frame * N;
            for (int t = 4 * pl; t < N; t += 4 * L)
                *reinterpret_cast<float4 *>(mine + t) = __ldg(reinterpret_cast<const float4 *>(g + t));
            ch = mine;
            __syncwarp();
        } else {
            ch = a.llr + (size_t)frame * N;
        }

        uint32_t pll = lp32; // LLR level pointers, levels T+1..tp
        uint64_t ppp = lp64; // partial-sum level pointers, levels T..n-1
        int P = grp_live ? 1 : 0;
        int ji = 0;
        float metric = 0.0f;
        uint32_t syn = 0u, cur = 0u, anc = (uint32_t)lane;

        int b_begin = 0;
        if (L == 32 && nb0 > 0 && grp_live) {
            // ---- frozen prefix (leaves [0, E), one path): decoded element-parallel by
            // the whole warp (s3::frozen_prefix; out of line so the block walk's code
            // generation is not disturbed)
            metric = frozen_prefix<FEX>(ch, llr, ps, n, tp, ss, psw, nb0 << T, a.metric_exact, lane);
            b_begin = nb0;
        }

        const int nblk = N >> T;
        for (int b = b_begin; b < nblk; ++b) {
            const int i0 = b << T;
            const bool act0 = pl < P;
            // ================= upper descent: level T into registers =================
            float x[BL];
            if (act0) {
                const int start = (b == 0) ? n - 1 : T + __ffs(b) - 1;
                if (start == T) {
                    // level T from level T+1 (read through the pointer, or the channel)
                    const float *src = (T + 1 == n) ? ch : llr + sl32(pll, T + 1) * ss + llo(T + 1);
                    const uint32_t g = (i0 >> T) & 1u;
                    const uint32_t bits = g ? ps[sl64(ppp, T) * psw + pso(T)] : 0u;
#pragma unroll
                    for (int t = 0; t < BL; t += 4) {
                        const float4 A = *reinterpret_cast<const float4 *>(src + t);
                        const float4 Bv = *reinterpret_cast<const float4 *>(src + BL + t);
                        const float4 o = g ? g4(A, Bv, bits >> t) : f4(A, Bv, FEX);
                        x[t] = o.x;
                        x[t + 1] = o.y;
                        x[t + 2] = o.z;
                        x[t + 3] = o.w;
                    }
                } else {
                    const int s0 = start < tp ? start : tp;
                    const int w0 = 1 << s0;
                    const uint32_t g0 = (i0 >> s0) & 1u;
                    float *dst = own + llo(s0);
                    const uint32_t *pw0 = ps + sl64(ppp, s0) * psw + pso(s0);
                    if (s0 + 1 <= tp) {
                        const float *src = llr + sl32(pll, s0 + 1) * ss + llo(s0 + 1);
                        if (g0)
                            level_from<FEX, true>(dst, src, w0, pw0);
                        else
                            level_from<FEX, false>(dst, src, w0, pw0);
                    } else if (NV == 0) {
                        if (g0)
                            level_from<FEX, true>(dst, ch, w0, pw0);
                        else
                            level_from<FEX, false>(dst, ch, w0, pw0);
                    } else {
                        if constexpr (NV > 0) {
                            const uint32_t *psp[NV];
                            uint32_t gm = 0;
#pragma unroll
                            for (int d = 0; d < NV; ++d) {
                                const int r = n - NV + d;
                                psp[d] = ps + sl64(ppp, r) * psw + pso(r);
                                gm |= ((uint32_t)(i0 >> r) & 1u) << d;
                            }
                            for (int t = 0; t < w0; t += 4) {
                                const float4 A = virt_top4<NV, FEX>(ch, n, t, psp, gm);
                                const float4 Bv = virt_top4<NV, FEX>(ch, n, t + w0, psp, gm);
                                *reinterpret_cast<float4 *>(dst + t) =
                                    g0 ? g4(A, Bv, pw0[t >> 5] >> (t & 31)) : f4(A, Bv, FEX);
                            }
                        }
                    }
                    for (int s = s0 - 1; s >= T + 1; --s)
                        level_from<FEX, false>(own + llo(s), own + llo(s + 1), 1 << s, nullptr);
                    const float *src = own + llo(T + 1);
#pragma unroll
                    for (int t = 0; t < BL; t += 4) {
                        const float4 o = f4(*reinterpret_cast<const float4 *>(src + t),
                                            *reinterpret_cast<const float4 *>(src + BL + t), FEX);
                        x[t] = o.x;
                        x[t + 1] = o.y;
                        x[t + 2] = o.z;
                        x[t + 3] = o.w;
                    }
                    for (int s = T + 1; s <= s0; ++s)
                        pll = set32(pll, s, lane); // levels T+1..s0 now live in the own slot
                }
            }
            __syncwarp();
            const uint32_t bmask = BL == 32 ? 0xffffffffu : ((1u << (BL & 31)) - 1u);
            const uint32_t fzw = (__ldg(frzg + (i0 >> 5)) >> (i0 & 31)) & bmask;
            const uint32_t daw = damg != nullptr ? (__ldg(damg + (i0 >> 5)) >> (i0 & 31)) & bmask : 0u;
            // the block's CRC syndrome columns, one per lane (a leaf takes its own by a
            // shuffle instead of a load on its decision chain)
#ifndef SCL3_COLB
#define SCL3_COLB 1
#endif
            const uint32_t colb = (SCL3_COLB && use_crc) ? __ldg(colg + i0 + (lane & (BL - 1))) : 0u;

            // ================= the block's leaves, registers only =================
            static_assert(T >= 3 && T <= 5, "the leaf code below is written for 8- to 32-leaf blocks");
            // registers of the block's levels below T (level T is x); unused ones for small T
            float l4[16], l3[8], l2[4], l1[2];
            uint32_t psr = 0;   // partial sums of levels < T: level s at bits [2^s - 1, 2^(s+1) - 1)
            uint32_t betaT = 0; // the block's codeword (2^T bits) after its last leaf
            // One copy of the leaf code for all leaves (runtime j, warp-uniform
            // branches): an unrolled block overflows the instruction cache.
#pragma unroll 1
            for (int j = 0; j < BL; ++j) {
                // ---- leaf descent: level ctz(j) by g, the levels below by f ----
                float lam;
                if (j & 1) {
                    lam = scl_g(l1[0], l1[1], psr & 1u);
                } else {
                    if (j & 2) {
                        l1[0] = scl_g(l2[0], l2[2], (psr >> 1) & 1u);
                        l1[1] = scl_g(l2[1], l2[3], (psr >> 2) & 1u);
                    } else {
                        const float *L3 = (T == 3) ? x : l3;
                        if (j & 4) {
#pragma unroll
                            for (int t = 0; t < 4; ++t)
                                l2[t] = scl_g(L3[t], L3[t + 4], (psr >> (3 + t)) & 1u);
                        } else {
                            if constexpr (T >= 4) {
                                const float *L4 = (T == 4) ? x : l4;
                                if (j & 8) {
#pragma unroll
                                    for (int t = 0; t < 8; ++t)
                                        l3[t] = scl_g(L4[t], L4[t + 8], (psr >> (7 + t)) & 1u);
                                } else {
                                    if constexpr (T >= 5) {
                                        if (j & 16) {
#pragma unroll
                                            for (int t = 0; t < 16; ++t)
                                                l4[t] = scl_g(x[t], x[t + 16], (psr >> (15 + t)) & 1u);
                                        } else {
#pragma unroll
                                            for (int t = 0; t < 16; ++t)
                                                l4[t] = scl_f<FEX>(x[t], x[t + 16]);
                                        }
                                    }
#pragma unroll
                                    for (int t = 0; t < 8; ++t)
                                        l3[t] = scl_f<FEX>(L4[t], L4[t + 8]);
                                }
                            }
#pragma unroll
                            for (int t = 0; t < 4; ++t)
                                l2[t] = scl_f<FEX>(L3[t], L3[t + 4]);
                        }
                        l1[0] = scl_f<FEX>(l2[0], l2[2]);
                        l1[1] = scl_f<FEX>(l2[1], l2[3]);
                    }
                    lam = scl_f<FEX>(l1[0], l1[1]);
                }
                const int i = i0 + j;
                const uint32_t fz = (fzw >> j) & 1u;
                const uint32_t dz = (daw >> j) & 1u;
                const bool act = pl < P;
                uint32_t col = 0u;
                if (!fz && use_crc)
                    col = SCL3_COLB ? __shfl_sync(FULL, colb, j) : __ldg(colg + i);
                float inc0, inc1;
                metric_incs(lam, CK ? true : (bool)a.metric_exact, inc0, inc1);
                uint32_t u = 0u;
                if (fz | dz) {
                    u = (dz && lam < 0.0f) ? 1u : 0u;
                    if (act)
                        metric += u ? inc1 : inc0;
                } else if constexpr (L == 1) {
                    // SC (one path per frame): keep the better child, a tie keeps u = 0
                    // (candidate index 0 < 1, _kernels.py:253-267); no slot moves
                    const float c0 = metric + inc0, c1 = metric + inc1;
                    u = c1 < c0 ? 1u : 0u;
                    if (act)
                        metric = u ? c1 : c0;
                } else {
                    const float c0 = act ? metric + inc0 : INFINITY;
                    const float c1 = act ? metric + inc1 : INFINITY;
                    bool k0 = act, k1 = act;
                    bool trivial = false; // full list, every path keeps its agreeing child
                    if (__any_sync(FULL, P == Lc)) {
                        // ---- selection at a full list: exactly the L best of 2L by (metric, index) ----
                        // (live groups share P; a finished group has P = 0 and takes no part)
                        // g = agreeing child, b = the other.  Every g below the best b is kept and
                        // every b above the worst g is dropped; the h = #{g >= min b} remaining
                        // slots go to the h smallest of the uncertain set U = {g >= min b} u {b <= max g}.
                        const bool z = c0 <= c1; // a tie keeps u = 0 (index p < L + p)
                        const float gv = z ? c0 : c1, bv = z ? c1 : c0;
                        const uint32_t gk = mkey(gv), bk = mkey(bv);
                        const int gi = z ? pl : L + pl, bi = z ? L + pl : pl;
                        const uint32_t gm = gmax_u<L>(act ? gk : 0u);
                        const uint32_t bm = gmin_u<L>(act ? bk : FULL);
                        const bool hiG = act && gk >= bm, loB = act && bk <= gm;
                        bool inG = act, inB = false;
                        S3_COUNT(0);
                        // (no g at or above the best b: the L agreeing children are the L best,
                        // no slot frees or clones -- 77% of the full-list selections, tools/scl3_stats.py)
#ifndef SCL3_TRIVIAL
#define SCL3_TRIVIAL 1
#endif
                        trivial = SCL3_TRIVIAL && !__any_sync(FULL, hiG);
                        if (trivial && act) {
                            u = z ? 0u : 1u;
                            metric = gv;
                        }
                        if (!trivial) {
                            S3_COUNT(1);
                            const uint32_t gb = (__ballot_sync(FULL, hiG) >> gbase) & gmask_lo;
                            const uint32_t bb = (__ballot_sync(FULL, loB) >> gbase) & gmask_lo;
                            const int h = __popc(gb), l = __popc(bb);
                            // (a group with some g >= min b has h >= 1 and l >= 1)
                            if (__all_sync(FULL, h <= 1 || l <= 1)) {
                                S3_COUNT(2);
                                // one swap at most: the worst kept g against the best dropped b
                                const int gx = gmax_i<L>(act && gk == gm ? gi : -1);
                                const int bx = gmin_i<L>(act && bk == bm ? bi : 2 * L);
                                if (h > 0 && (bm < gm || (bm == gm && bx < gx))) {
                                    if (gk == gm && gi == gx)
                                        inG = false;
                                    if (bk == bm && bi == bx)
                                        inB = true;
                                }
                            } else {
                                // rank inside U by (metric, index): strict metric ranks first,
                                // the exact key only when U holds tied metrics (rank sum check)
                                const uint32_t below = (1u << pl) - 1u;
                                const int nu = h + l;
                                float *um = cg;                                 // U metrics
                                int *ui = reinterpret_cast<int *>(cg + 2 * L);  // U candidate indices
                                const int qg = __popc(gb & below), qb = h + __popc(bb & below);
                                if (hiG) {
                                    um[qg] = gv;
                                    ui[qg] = gi;
                                }
                                if (loB) {
                                    um[qb] = bv;
                                    ui[qb] = bi;
                                }
                                int rg = 0, rb = 0;
                                if constexpr (L == 32) {
                                    // one group: nu is warp-uniform; pad U to a multiple of 4 with +inf
                                    if (lane < ((-nu) & 3))
                                        um[nu + lane] = INFINITY;
                                    __syncwarp();
                                    for (int q = 0; q < nu; q += 4) {
                                        const float4 v = *reinterpret_cast<const float4 *>(um + q);
                                        rg += (v.x < gv) + (v.y < gv) + (v.z < gv) + (v.w < gv);
                                        rb += (v.x < bv) + (v.y < bv) + (v.z < bv) + (v.w < bv);
                                    }
                                } else {
                                    if (nu & 1)
                                        um[nu] = INFINITY; // pad to pairs
                                    __syncwarp();
                                    const int numax = __reduce_max_sync(FULL, nu);
                                    for (int q = 0; q < numax; q += 2) {
                                        const float2 v = *reinterpret_cast<const float2 *>(um + q);
                                        const bool l0 = q < nu, l1v = q + 1 < nu;
                                        rg += (l0 && v.x < gv) + (l1v && v.y < gv);
                                        rb += (l0 && v.x < bv) + (l1v && v.y < bv);
                                    }
                                }
                                // no ties inside U <=> the strict ranks of its nu elements sum to nu(nu-1)/2
                                const int rsum = gsum_i<L>((hiG ? rg : 0) + (loB ? rb : 0));
                                if (__any_sync(FULL, rsum != nu * (nu - 1) / 2)) {
                                    rg = 0;
                                    rb = 0;
                                    const int numax2 = __reduce_max_sync(FULL, nu);
                                    for (int q = 0; q < numax2; ++q) {
                                        const float v = um[q];
                                        const int vi = ui[q];
                                        const bool live = q < nu;
                                        rg += live && (v < gv || (v == gv && vi < gi));
                                        rb += live && (v < bv || (v == bv && vi < bi));
                                    }
                                }
                                if (hiG)
                                    inG = rg < h;
                                if (loB)
                                    inB = rb < h;
                                __syncwarp();
                            }
                        }
                        k0 = z ? inG : inB;
                        k1 = z ? inB : inG;
                    } else if (__any_sync(FULL, 2 * P > Lc)) {
                        // growth past a list size that is not a power of two (P < Lc < 2P):
                        // keep the Lc smallest of the 2P candidates by (metric, index),
                        // the candidate index of the u = 1 child being Lc + p (_kernels.py:253-267)
                        float *um = cg;
                        int *ui = reinterpret_cast<int *>(cg + 2 * L);
                        if (act) {
                            um[pl] = c0;
                            ui[pl] = pl;
                            um[P + pl] = c1;
                            ui[P + pl] = Lc + pl;
                        }
                        __syncwarp();
                        int r0 = 0, r1 = 0;
                        for (int q = 0; q < 2 * P; ++q) {
                            const float v = um[q];
                            const int vi = ui[q];
                            r0 += v < c0 || (v == c0 && vi < pl);
                            r1 += v < c1 || (v == c1 && vi < Lc + pl);
                        }
                        k0 = act && r0 < Lc;
                        k1 = act && r1 < Lc;
                        __syncwarp();
                    }
                    // ---- slot assignment (_kernels.py:271-311) ----
                    if (!trivial) {
                    const uint32_t freeM = (__ballot_sync(FULL, act && !k0 && !k1) >> gbase) & gmask_lo;
                    const uint32_t dupM = (__ballot_sync(FULL, act && k0 && k1) >> gbase) & gmask_lo;
                    const int nf = __popc(freeM), nd = __popc(dupM);
                    int src = lane;
                    // the r-th free slot (freed lanes, then virgin lanes) clones the r-th
                    // duplicating parent: parents post their lane in a rank table
                    int *ptab = reinterpret_cast<int *>(cg);
                    const bool anydup = __any_sync(FULL, nd > 0);
                    if (anydup) {
                        if (act && k0 && k1)
                            ptab[__popc(dupM & ((1u << pl) - 1u))] = lane;
                        __syncwarp();
                    }
                    if (act && (k0 || k1)) {
                        u = k0 ? 0u : 1u;
                        metric = k0 ? c0 : c1;
                    } else {
                        const int r = act ? __popc(freeM & ((1u << pl) - 1u)) : nf + (pl - P);
                        if (r < nd)
                            src = ptab[r];
                    }
                    if (anydup)
                        __syncwarp();
                    if (__any_sync(FULL, src != lane)) {
                        S3_COUNT(3);
                        const float pc1 = __shfl_sync(FULL, c1, src);
                        // eager copy of the still-readable register levels: level s+1 while
                        // bit s of j is 0 (the reference's rule at _kernels.py:296-303)
                        if (((j >> (T - 1)) & 1) == 0) {
#pragma unroll
                            for (int t = 0; t < BL; ++t)
                                x[t] = __shfl_sync(FULL, x[t], src);
                        }
                        if (T >= 5 && (j & 8) == 0) {
#pragma unroll
                            for (int t = 0; t < 16; ++t)
                                l4[t] = __shfl_sync(FULL, l4[t], src);
                        }
                        if (T >= 4 && (j & 4) == 0) {
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                l3[t] = __shfl_sync(FULL, l3[t], src);
                        }
                        if ((j & 2) == 0) {
#pragma unroll
                            for (int t = 0; t < 4; ++t)
                                l2[t] = __shfl_sync(FULL, l2[t], src);
                        }
                        if ((j & 1) == 0) {
                            l1[0] = __shfl_sync(FULL, l1[0], src);
                            l1[1] = __shfl_sync(FULL, l1[1], src);
                        }
                        const uint32_t psr2 = __shfl_sync(FULL, psr, src);
                        const uint32_t pll2 = __shfl_sync(FULL, pll, src);
                        const uint32_t pp_lo = __shfl_sync(FULL, (uint32_t)ppp, src);
                        const uint32_t pp_hi = __shfl_sync(FULL, (uint32_t)(ppp >> 32), src);
                        const uint32_t syn2 = __shfl_sync(FULL, syn, src);
                        const uint32_t cur2 = __shfl_sync(FULL, cur, src);
                        const uint32_t anc2 = __shfl_sync(FULL, anc, src);
                        if (src != lane) {
                            u = 1u;
                            metric = pc1;
                            psr = psr2;
                            pll = pll2;
                            ppp = ((uint64_t)pp_hi << 32) | pp_lo;
                            syn = syn2;
                            cur = cur2;
                            anc = anc2;
                        }
                    }
                    P = P == 0 ? 0 : P - nf + nd;
                    }
                }
                // ---- record the decision (non-frozen positions) ----
                if (!fz) {
                    cur |= u << (ji & 31);
                    syn ^= u ? col : 0u;
                    ++ji;
                    if ((ji & 31) == 0) {
                        const int w = (ji >> 5) - 1;
                        tb[w * 32 + lane] = cur;
                        tba[w * 32 + lane] = (uint8_t)anc;
                        cur = 0u;
                        anc = (uint32_t)lane;
                    }
                }
                // ---- fold u into the register partial sums: level S = trailing ones of j ----
                {
                    uint32_t Fw = u;
                    if (j & 1) {
                        Fw = ((psr ^ Fw) & 1u) | (Fw << 1);
                        if (j & 2) {
                            Fw = (((psr >> 1) ^ Fw) & 3u) | (Fw << 2);
                            if (j & 4) {
                                Fw = (((psr >> 3) ^ Fw) & 15u) | (Fw << 4);
                                if constexpr (T == 3) {
                                    betaT = Fw;
                                } else {
                                    if (j & 8) {
                                        Fw = (((psr >> 7) ^ Fw) & 255u) | (Fw << 8);
                                        if constexpr (T == 4) {
                                            betaT = Fw;
                                        } else {
                                            if (j & 16)
                                                betaT = (((psr >> 15) ^ Fw) & 0xffffu) | (Fw << 16);
                                            else
                                                psr = (psr & ~(0xffffu << 15)) | (Fw << 15);
                                        }
                                    } else {
                                        psr = (psr & ~(255u << 7)) | (Fw << 7);
                                    }
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
            }

            // ================= block end: fold the block codeword into the shared levels =================
            if (pl < P) {
                const int S = T + __ffs(~b) - 1; // level of the node completed by this block
                if (S < n) {
                    uint32_t F5 = betaT;
                    const int lo = S < 5 ? S : 5;
                    for (int s = T; s < lo; ++s) {
                        const int len = 1 << s;
                        const uint32_t pv = ps[sl64(ppp, s) * psw + pso(s)];
                        F5 = ((pv ^ F5) & ((1u << len) - 1u)) | (F5 << len);
                    }
                    uint32_t *dst = pown + pso(S);
                    if (S <= 5) {
                        dst[0] = F5;
                    } else {
                        const int words = 1 << (S - 5);
                        for (int w = 0; w < words; ++w) {
                            uint32_t v = F5;
                            for (int s = 5; s < S; ++s)
                                if (((w >> (s - 5)) & 1) == 0)
                                    v ^= ps[sl64(ppp, s) * psw + pso(s) + (w & ((1 << (s - 5)) - 1))];
                            dst[w] = v;
                        }
                    }
                    ppp = set64(ppp, S, lane);
                }
            }
            __syncwarp();
        }
        if ((ji & 31) != 0) {
            const int w = ji >> 5;
            tb[w * 32 + lane] = cur;
            tba[w * 32 + lane] = (uint8_t)anc;
        }

        // ---- winner: least (metric, slot) among CRC-passing paths (scl.py:177-191) ----
        const bool act = pl < P;
        const bool ok = act && use_crc && syn == a.code.crc_offset;
        const uint32_t okM = (__ballot_sync(FULL, ok) >> gbase) & gmask_lo;
        const bool cnd = okM ? ok : act;
        float key = cnd ? metric : INFINITY;
        int who = cnd ? pl : L;
#pragma unroll
        for (int off = 1; off < L; off <<= 1) {
            const float k2 = __shfl_xor_sync(FULL, key, off);
            const int w2 = __shfl_xor_sync(FULL, who, off);
            if (k2 < key || (k2 == key && w2 < who)) {
                key = k2;
                who = w2;
            }
        }
        __syncwarp();
        if (grp_live && pl == 0) {
            // traceback of the winner's decision windows
            int l = gbase + who;
            for (int w = W - 1; w >= 0; --w) {
                wrow[grp * W + w] = tb[w * 32 + l];
                l = gbase + (tba[w * 32 + l] - gbase);
            }
        }
        __syncwarp();
        if (grp_live) {
            const uint32_t *row = wrow + grp * W;
            const int NW = (N + 31) >> 5;
            if (a.u_bits != nullptr)
                for (int w = pl; w < NW; w += L) {
                    int rank = 0;
                    for (int z = 0; z < w; ++z)
                        rank += 32 - __popc(__ldg(frzg + z));
                    const uint32_t fw = __ldg(frzg + w);
                    uint32_t v = 0;
                    for (int q = 0; q < 32 && 32 * w + q < N; ++q)
                        if (!((fw >> q) & 1u)) {
                            v |= ((row[rank >> 5] >> (rank & 31)) & 1u) << q;
                            ++rank;
                        }
                    a.u_bits[(size_t)frame * NW + w] = v;
                }
            if (a.payload != nullptr) {
                const int MW = (a.code.m + 31) >> 5;
                for (int w = pl; w < MW; w += L) {
                    uint32_t v = row[w];
                    if (32 * w + 32 > a.code.m)
                        v &= (1u << (a.code.m & 31)) - 1u;
                    a.payload[(size_t)frame * MW + w] = v;
                }
            }
            if (pl == 0) {
                if (a.metric != nullptr)
                    a.metric[frame] = key;
                if (a.crc_ok != nullptr)
                    a.crc_ok[frame] = okM != 0;
                if (a.sel != nullptr)
                    a.sel[frame] = okM != 0;
                if (a.t_done != nullptr)
                    a.t_done[frame] = globaltimer();
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------- launchers --


template <int CN, int NV, int L>
inline bool scl3_geom_is(const SclArgs &a)
{
    using G = Scl3Geom<CN, NV>;
    if (a.code.n != CN || a.tp != G::tp || a.ss != G::ss || a.psw != G::psw)
        return false;
    // the default knobs the compiled-in kernels also fix: exact metric, CRC on,
    // no decision-aided positions, channel from global memory, a full
    // power-of-two list, the frozen-prefix path at L = 32
    return !SCL3_CN_ME || (a.metric_exact && a.code.crc_width > 0 && a.code.da_bits == nullptr && a.o_ch < 0 &&
                           (a.list_cap <= 0 || a.list_cap >= L) && (L != 32 || a.prefix));
}

template <int L, bool FEX, int NV>
inline int launch_scl3_t(const SclArgs &a, int wpc, int max_warps, cudaStream_t s)
{
    auto kern = k_scl3<L, FEX, NV>;
    // the default list decoders at N = 1024..4096 (min-sum f, 3 virtual levels)
    // with the geometry compiled in (+5% at N = 1024, L = 32)
    if constexpr (SCL3_CN && !FEX && NV == 3) {
        switch (a.code.n) {
        case 10:
            if (scl3_geom_is<10, NV, L>(a))
                kern = k_scl3<L, FEX, NV, 10>;
            break;
        case 11:
            if (scl3_geom_is<11, NV, L>(a))
                kern = k_scl3<L, FEX, NV, 11>;
            break;
        case 12:
            if (scl3_geom_is<12, NV, L>(a))
                kern = k_scl3<L, FEX, NV, 12>;
            break;
        }
    }
    const size_t per_warp = (size_t)a.warp_words * 4;
    const size_t smem_cap = 227 * 1024;
    if (per_warp > smem_cap)
        return PC_ERR_UNSUPPORTED;
    while (wpc > 1 && (size_t)wpc * per_warp > smem_cap)
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
    const long long need = ((long long)max_warps + wpc - 1) / wpc;
    if (grid > need)
        grid = need;
    if (grid < 1)
        grid = 1;
    kern<<<(int)grid, 32 * wpc, smem, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

template <int L, bool FEX>
inline int launch_scl3_nv(const SclArgs &a, int wpc, int max_warps, cudaStream_t s)
{
    switch (a.nv) {
    case 0: return launch_scl3_t<L, FEX, 0>(a, wpc, max_warps, s);
    case 1: return launch_scl3_t<L, FEX, 1>(a, wpc, max_warps, s);
    case 2: return launch_scl3_t<L, FEX, 2>(a, wpc, max_warps, s);
    case 3: return launch_scl3_t<L, FEX, 3>(a, wpc, max_warps, s);
    case 4: return launch_scl3_t<L, FEX, 4>(a, wpc, max_warps, s);
    default: return PC_ERR_UNSUPPORTED;
    }
}

// One translation unit per list size (scl3_l*.cu) instantiates this, so the
// 60 kernel variants compile in parallel.
template <int L>
int launch_scl3_for(const SclArgs &a, int wpc, int max_warps, cudaStream_t s)
{
    return a.f_exact ? launch_scl3_nv<L, true>(a, wpc, max_warps, s) : launch_scl3_nv<L, false>(a, wpc, max_warps, s);
}

} // namespace pc
