// scl.cu -- K3: CRC-aided successive-cancellation list decoding (sm_100a).
//
// Restates _kernels.scl_decode_kernel (reference _kernels.py:144-333) and the
// winner rule of scl.scl_decode (scl.py:177-191) with the same LOGICAL slot
// numbering, so ties resolve exactly as in the reference:
//   * candidate index p for u = 0, L + p for u = 1         (_kernels.py:247-249)
//   * survivors = up to L best by (metric, candidate index) (_kernels.py:253-267)
//   * u = 0 child keeps the slot, else the u = 1 child; a parent with no
//     surviving child frees its slot                        (_kernels.py:271-281)
//   * duplicates fill freed slots in ascending parent order, then virgin
//     slots                                                 (_kernels.py:285-311)
//   * winner = least (metric, slot) among CRC-passing paths (scl.py:181-191)
//
// Mapping (B200-first, not the reference's loop nest):
//   * one WARP decodes F = 32 / L frames; lane = (frame group, path) and the
//     lane index IS the physical slot of that logical path.  Every f/g level
//     is a per-lane loop over that path's elements, so the whole decoder runs
//     with __syncwarp only -- no CTA barriers, 32 paths in SIMT lock-step;
//   * path copies are LAZY: each lane keeps, in two 64-bit registers, a 5-bit
//     slot pointer per tree level (LLR levels and partial-sum levels).  A
//     clone copies its parent's pointers (two shuffles) instead of the data;
//     writes always go to the lane's own slot.  Because all paths rewrite the
//     same levels at the same bit index, a level is never overwritten while
//     another path still points to it ("SCL lazy copies");
//   * the top `NV` tree levels are not stored: they are recomputed from the
//     channel LLRs when the highest stored level needs them, which cuts shared
//     memory per warp (and raises warps per SM) at a small FMA cost;
//   * survivor selection is a pairwise rank count over the group's 2L
//     candidates with warp shuffles; slot assignment uses ballots.
#include "args.cuh"

namespace pc {


__device__ __forceinline__ float f_minsum(float a, float b)
{
    // _kernels.py:40-48: zero if either input is zero, else sign * min
    float mag = fminf(fabsf(a), fabsf(b));
    if ((a < 0.0f) != (b < 0.0f))
        mag = -mag;
    return (a == 0.0f || b == 0.0f) ? 0.0f : mag;
}

__device__ __forceinline__ float f_boxplus(float a, float b)
{
    // _kernels.py:51-65
    const float s = a + b;
    const float num = s > 0.0f ? s + log1pf(expf(-s)) : log1pf(expf(s));
    const float den = a >= b ? a + log1pf(expf(b - a)) : b + log1pf(expf(a - b));
    return num - den;
}

template <bool FEX>
__device__ __forceinline__ float scl_f(float a, float b)
{
    return FEX ? f_boxplus(a, b) : f_minsum(a, b);
}

__device__ __forceinline__ float scl_g(float a, float b, uint32_t u) { return u ? b - a : b + a; }

// Metric increments for both decisions at soft value lam (_kernels.py:76-90).
__device__ __forceinline__ void metric_incs(float lam, bool exact, float &inc0, float &inc1)
{
    if (exact) {
        const float y = fabsf(lam);
        const float sp = log1pf(expf(-y));
        const float agree = sp, disagree = y + sp;
        // x = lam for u = 0: x > 0 -> sp(x); x <= 0 -> -x + sp(-x)
        inc0 = lam > 0.0f ? agree : disagree;
        inc1 = lam < 0.0f ? agree : disagree;
        if (lam == 0.0f)
            inc0 = inc1 = sp;
    } else {
        inc0 = lam < 0.0f ? -lam : 0.0f;
        inc1 = lam > 0.0f ? lam : 0.0f;
    }
}

// word offset of partial-sum level s: levels < 5 take one word, level s >= 5 takes 2^(s-5)
__host__ __device__ __forceinline__ int ps_off(int s) { return s <= 5 ? s : (1 << (s - 5)) + 4; }

__device__ __forceinline__ int slot_of(uint64_t ptrs, int s) { return (int)((ptrs >> (5 * s)) & 31u); }
__device__ __forceinline__ uint64_t set_slot(uint64_t ptrs, int s, int v)
{
    return (ptrs & ~(31ull << (5 * s))) | ((uint64_t)v << (5 * s));
}

// Per-lane view of the tree: pointer registers and the recomputed top levels.
struct Tree {
    const float *ch;    // channel LLRs of this lane's frame
    const uint32_t *ps; // warp partial-sum slots
    int n, i, psw;
    uint64_t pl, pp; // pointer registers (llr levels, partial-sum levels)

    __device__ __forceinline__ uint32_t psbit(int s, int t) const
    {
        return (ps[slot_of(pp, s) * psw + ps_off(s) + (t >> 5)] >> (t & 31)) & 1u;
    }

    // Recompute element t of the highest virtual level s = n - NV from the
    // 2^NV channel leaves t + j 2^s (bottom-up, registers only).
    template <int NV, bool FEX>
    __device__ __forceinline__ float virt(int t) const
    {
        static_assert(NV >= 1 && NV <= 4, "virtual levels");
        constexpr int CNT = 1 << (NV - 1);
        const int s = n - NV;
        const int half = 1 << (n - 1);
        float v[CNT];
        const bool g_top = (i >> (n - 1)) & 1;
#pragma unroll
        for (int j = 0; j < CNT; ++j) {
            const int x = t + (j << s);
            const float A = __ldg(ch + x), B = __ldg(ch + x + half);
            v[j] = g_top ? scl_g(A, B, psbit(n - 1, x)) : scl_f<FEX>(A, B);
        }
#pragma unroll
        for (int d = NV - 2; d >= 0; --d) { // level r = s + d, d counts down to s
            const int r = s + d;
            const int c = 1 << d;
            const bool g = (i >> r) & 1;
#pragma unroll
            for (int j = 0; j < c; ++j) {
                const int x = t + (j << s);
                v[j] = g ? scl_g(v[j], v[j + c], psbit(r, x)) : scl_f<FEX>(v[j], v[j + c]);
            }
        }
        return v[0];
    }
};

template <int L, bool FEX, int NV>
__global__ void __launch_bounds__(128) k_scl(const SclArgs a)
{
    constexpr int F = 32 / L;
    extern __shared__ __align__(16) uint32_t smw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    uint32_t *wbase = smw + (size_t)wib * a.warp_words;
    float *llr = reinterpret_cast<float *>(wbase);
    uint32_t *ps = wbase + 32 * a.ss;
    uint32_t *uh = ps + 32 * a.psw;

    const int n = a.code.n, N = a.code.N, tp = a.tp;
    const int grp = lane / L, gbase = grp * L, pl = lane - gbase;
    const uint32_t gmask_lo = (L == 32) ? 0xffffffffu : ((1u << L) - 1u);
    const int total = a.count != nullptr ? *a.count : a.B;
    const int NW = (N + 31) >> 5;

    for (;;) {
        int base = 0;
        if (lane == 0)
            base = atomicAdd(a.work, F);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= total)
            break;
        const int qi = base + grp;
        const bool grp_live = qi < total;
        const int frame = grp_live ? (a.queue != nullptr ? a.queue[qi] : qi) : 0;

        Tree T;
        T.ch = a.llr + (size_t)frame * N;
        T.ps = ps;
        T.n = n;
        T.psw = a.psw;
        T.pl = 0;
        T.pp = 0;
        for (int s = 0; s < 12; ++s) {
            T.pl = set_slot(T.pl, s, lane);
            T.pp = set_slot(T.pp, s, lane);
        }
        int P = grp_live ? 1 : 0;
        float metric = 0.0f;
        float *own = llr + lane * a.ss;

        for (int i = 0; i < N; ++i) {
            T.i = i;
            const bool act = pl < P;
            // ---- descent: levels min(start, tp) .. 0 ----
            if (act) {
                const int start = (i == 0) ? n - 1 : __ffs(i) - 1;
                for (int s = start < tp ? start : tp; s >= 0; --s) {
                    const int w = 1 << s;
                    const bool gop = (i >> s) & 1;
                    float *dst = own + w;
                    if (s + 1 <= tp) {
                        const float *src = llr + slot_of(T.pl, s + 1) * a.ss + 2 * w;
                        const uint32_t *pw = ps + slot_of(T.pp, s) * a.psw + ps_off(s);
                        if (w >= 4) {
                            for (int t = 0; t < w; t += 4) {
                                const float4 A = *reinterpret_cast<const float4 *>(src + t);
                                const float4 B = *reinterpret_cast<const float4 *>(src + w + t);
                                float4 o;
                                if (gop) {
                                    const uint32_t bits = pw[t >> 5] >> (t & 31);
                                    o.x = scl_g(A.x, B.x, bits & 1u);
                                    o.y = scl_g(A.y, B.y, (bits >> 1) & 1u);
                                    o.z = scl_g(A.z, B.z, (bits >> 2) & 1u);
                                    o.w = scl_g(A.w, B.w, (bits >> 3) & 1u);
                                } else {
                                    o.x = scl_f<FEX>(A.x, B.x);
                                    o.y = scl_f<FEX>(A.y, B.y);
                                    o.z = scl_f<FEX>(A.z, B.z);
                                    o.w = scl_f<FEX>(A.w, B.w);
                                }
                                *reinterpret_cast<float4 *>(dst + t) = o;
                            }
                        } else {
                            for (int t = 0; t < w; ++t) {
                                const float A = src[t], B = src[w + t];
                                dst[t] = gop ? scl_g(A, B, (pw[0] >> t) & 1u) : scl_f<FEX>(A, B);
                            }
                        }
                    } else if (s + 1 == n) {
                        // level n-1 straight from the channel (no virtual levels)
                        const uint32_t *pw = ps + slot_of(T.pp, s) * a.psw + ps_off(s);
                        for (int t = 0; t < w; ++t) {
                            const float A = __ldg(T.ch + t), B = __ldg(T.ch + w + t);
                            dst[t] = gop ? scl_g(A, B, (pw[t >> 5] >> (t & 31)) & 1u) : scl_f<FEX>(A, B);
                        }
                    } else {
                        const uint32_t *pw = ps + slot_of(T.pp, s) * a.psw + ps_off(s);
                        for (int t = 0; t < w; ++t) {
                            float A = 0.0f, B = 0.0f;
                            if constexpr (NV > 0) {
                                A = T.virt<NV, FEX>(t);
                                B = T.virt<NV, FEX>(t + w);
                            }
                            dst[t] = gop ? scl_g(A, B, (pw[t >> 5] >> (t & 31)) & 1u) : scl_f<FEX>(A, B);
                        }
                    }
                    T.pl = set_slot(T.pl, s, lane);
                }
            }
            __syncwarp();
            const float lam = act ? own[1] : 0.0f;
            const bool frz = bit_of(a.code.frozen_bits, i);
            const bool da = !frz && a.code.da_bits != nullptr && bit_of(a.code.da_bits, i);
            uint32_t u = 0;
            bool newact = act;
            if (frz || da) {
                float inc0, inc1;
                metric_incs(lam, a.metric_exact, inc0, inc1);
                u = (da && lam < 0.0f) ? 1u : 0u;
                if (act)
                    metric += u ? inc1 : inc0;
            } else {
                // ---- branch: 2L candidates, keep the L best by (metric, index) ----
                float inc0, inc1;
                metric_incs(lam, a.metric_exact, inc0, inc1);
                const float c0 = act ? metric + inc0 : INFINITY;
                const float c1 = act ? metric + inc1 : INFINITY;
                bool k0 = act, k1 = act;
                if (__any_sync(0xffffffffu, 2 * P > L)) {
                    int r0 = 0, r1 = 0;
#pragma unroll
                    for (int q = 0; q < L; ++q) {
                        const float v0 = __shfl_sync(0xffffffffu, c0, gbase + q);
                        const float v1 = __shfl_sync(0xffffffffu, c1, gbase + q);
                        r0 += (v0 < c0 || (v0 == c0 && q <= pl)) + (v1 < c0);
                        r1 += (v0 <= c1) + (v1 < c1 || (v1 == c1 && q <= pl));
                    }
                    k0 = act && r0 <= L && c0 < INFINITY;
                    k1 = act && r1 <= L && c1 < INFINITY;
                }
                const uint32_t freeM = (__ballot_sync(0xffffffffu, act && !k0 && !k1) >> gbase) & gmask_lo;
                const uint32_t dupM = (__ballot_sync(0xffffffffu, act && k0 && k1) >> gbase) & gmask_lo;
                const int nf = __popc(freeM), nd = __popc(dupM);
                const bool surv = act && (k0 || k1);
                int src = lane;
                if (surv) {
                    u = k0 ? 0u : 1u;
                    metric = k0 ? c0 : c1;
                } else {
                    const int r = act ? __popc(freeM & ((1u << pl) - 1u)) : nf + (pl - P);
                    if (pl < L && r < nd) {
                        // r-th set bit of dupM = the parent this slot clones
                        uint32_t m = dupM;
                        for (int z = 0; z < r; ++z)
                            m &= m - 1u;
                        src = gbase + __ffs(m) - 1;
                    }
                }
                const bool clone = src != lane;
                const float pc1 = __shfl_sync(0xffffffffu, c1, src);
                const uint32_t pl_lo = __shfl_sync(0xffffffffu, (uint32_t)T.pl, src);
                const uint32_t pl_hi = __shfl_sync(0xffffffffu, (uint32_t)(T.pl >> 32), src);
                const uint32_t pp_lo = __shfl_sync(0xffffffffu, (uint32_t)T.pp, src);
                const uint32_t pp_hi = __shfl_sync(0xffffffffu, (uint32_t)(T.pp >> 32), src);
                if (clone) {
                    u = 1u;
                    metric = pc1;
                    T.pl = ((uint64_t)pl_hi << 32) | pl_lo;
                    T.pp = ((uint64_t)pp_hi << 32) | pp_lo;
                    const uint32_t *from = uh + src * a.uhs;
                    uint32_t *to = uh + lane * a.uhs;
                    for (int w = 0; w <= (i >> 5); ++w)
                        to[w] = from[w];
                }
                newact = surv || clone;
                P = P == 0 ? 0 : P - nf + nd;
                __syncwarp();
            }
            if (newact) {
                // record the decision, then fold it into the partial sums
                uint32_t *row = uh + lane * a.uhs;
                const uint32_t bm = 1u << (i & 31);
                row[i >> 5] = u ? (row[i >> 5] | bm) : (row[i >> 5] & ~bm);
                int S = __ffs(~i) - 1; // trailing ones of i
                if (S < n) {
                    uint32_t F5 = u ? 1u : 0u;
                    const int lo = S < 5 ? S : 5;
                    for (int s = 0; s < lo; ++s) {
                        const int len = 1 << s;
                        const uint32_t pv = ps[slot_of(T.pp, s) * a.psw + ps_off(s)];
                        const uint32_t msk = (len == 32) ? 0xffffffffu : ((1u << len) - 1u);
                        F5 = ((pv ^ F5) & msk) | (F5 << len);
                    }
                    uint32_t *dst = ps + lane * a.psw + ps_off(S);
                    if (S <= 5) {
                        dst[0] = F5;
                    } else {
                        const int words = 1 << (S - 5);
                        for (int w = 0; w < words; ++w) {
                            uint32_t v = F5;
                            for (int s = 5; s < S; ++s)
                                if (((w >> (s - 5)) & 1) == 0)
                                    v ^= ps[slot_of(T.pp, s) * a.psw + ps_off(s) + (w & ((1 << (s - 5)) - 1))];
                            dst[w] = v;
                        }
                    }
                    T.pp = set_slot(T.pp, S, lane);
                }
            }
            __syncwarp();
        }

        // ---- winner: least (metric, slot) among CRC-passing paths (scl.py:177-191) ----
        const bool act = pl < P;
        bool ok = false;
        if (act && a.code.crc_width > 0) {
            uint32_t syn = 0;
            const uint32_t *row = uh + lane * a.uhs;
            for (int w = 0; w < NW; ++w) {
                uint32_t v = row[w];
                if (32 * w + 32 > N)
                    v &= (1u << (N & 31)) - 1u;
                while (v) {
                    const int b = __ffs(v) - 1;
                    v &= v - 1u;
                    syn ^= __ldg(a.code.crc_cols + 32 * w + b);
                }
            }
            ok = syn == a.code.crc_offset;
        }
        const uint32_t okM = (__ballot_sync(0xffffffffu, ok) >> gbase) & gmask_lo;
        const bool cand = okM ? ok : act;
        float key = cand ? metric : INFINITY;
        int who = cand ? pl : L;
#pragma unroll
        for (int off = 1; off < L; off <<= 1) {
            const float k2 = __shfl_xor_sync(0xffffffffu, key, off);
            const int w2 = __shfl_xor_sync(0xffffffffu, who, off);
            if (k2 < key || (k2 == key && w2 < who)) {
                key = k2;
                who = w2;
            }
        }
        if (grp_live) {
            const uint32_t *row = uh + (gbase + who) * a.uhs;
            if (a.u_bits != nullptr)
                for (int w = pl; w < NW; w += L) {
                    uint32_t v = row[w];
                    if (32 * w + 32 > N)
                        v &= (1u << (N & 31)) - 1u;
                    a.u_bits[(size_t)frame * NW + w] = v;
                }
            if (a.payload != nullptr) {
                const int MW = (a.code.m + 31) >> 5;
                for (int w = pl; w < MW; w += L) {
                    uint32_t v = 0;
                    for (int b = 0; b < 32 && 32 * w + b < a.code.m; ++b)
                        v |= bit_of(row, __ldg(a.code.info_pos + 32 * w + b)) << b;
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


int scl_prepare(SclArgs &a, int nv_req)
{
    const int n = a.code.n;
    int nv = nv_req;
    if (nv < 0)
        nv = 0;
    if (nv > n - 1)
        nv = n - 1;
    if (nv > 3)
        nv = 3;
    a.nv = nv;
    a.tp = n - 1 - nv;
    a.ss = (1 << (a.tp + 1)) + 4;
    a.psw = ps_off(n) | 1; // words for levels 0..n-1, odd stride
    const int nw = (a.code.N + 31) >> 5;
    a.uhs = nw | 1;
    a.warp_words = 32 * (a.ss + a.psw + a.uhs);
    return PC_OK;
}

template <int L, bool FEX, int NV>
static int launch_scl_t(const SclArgs &a, int wpc, int max_warps, cudaStream_t s)
{
    auto kern = k_scl<L, FEX, NV>;
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
static int launch_scl_nv(const SclArgs &a, int wpc, int max_warps, cudaStream_t s)
{
    switch (a.nv) {
    case 0: return launch_scl_t<L, FEX, 0>(a, wpc, max_warps, s);
    case 1: return launch_scl_t<L, FEX, 1>(a, wpc, max_warps, s);
    case 2: return launch_scl_t<L, FEX, 2>(a, wpc, max_warps, s);
    case 3: return launch_scl_t<L, FEX, 3>(a, wpc, max_warps, s);
    default: return PC_ERR_UNSUPPORTED;
    }
}

template <bool FEX>
static int launch_scl_f(const SclArgs &a, int L, int wpc, int max_warps, cudaStream_t s)
{
    switch (L) {
    case 1: return launch_scl_nv<1, FEX>(a, wpc, max_warps, s);
    case 2: return launch_scl_nv<2, FEX>(a, wpc, max_warps, s);
    case 4: return launch_scl_nv<4, FEX>(a, wpc, max_warps, s);
    case 8: return launch_scl_nv<8, FEX>(a, wpc, max_warps, s);
    case 16: return launch_scl_nv<16, FEX>(a, wpc, max_warps, s);
    case 32: return launch_scl_nv<32, FEX>(a, wpc, max_warps, s);
    default: return PC_ERR_UNSUPPORTED;
    }
}

int launch_scl(const SclArgs &a, int L, int wpc, cudaStream_t s)
{
    if (a.B == 0)
        return PC_OK;
    if (cudaMemsetAsync(a.work, 0, sizeof(int32_t), s) != cudaSuccess)
        return PC_ERR_CUDA;
    const int F = 32 / L;
    const int max_warps = (a.B + F - 1) / F;
    if (wpc < 1 || wpc > 4)
        wpc = 1;
    return a.f_exact ? launch_scl_f<true>(a, L, wpc, max_warps, s) : launch_scl_f<false>(a, L, wpc, max_warps, s);
}

} // namespace pc
