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
//     is a per-lane loop over that path's elements (float4 shared-memory
//     traffic), so the decoder synchronises with __syncwarp only -- no CTA
//     barriers, L paths in SIMT lock-step;
//   * path copies are LAZY: each lane keeps, in two 64-bit registers, a 5-bit
//     slot pointer per tree level (LLR levels and partial-sum levels).  A
//     clone copies its parent's pointers (shuffles) instead of the data;
//     writes always go to the lane's own slot.  Because all paths rewrite the
//     same levels at the same bit index, a level is never overwritten while
//     another path still points to it ("SCL lazy copies");
//   * the top NV tree levels are not stored but recomputed from the channel
//     LLRs (kept in shared memory for L >= 16) when the highest stored level
//     needs them: less shared memory per warp, more warps per SM;
//   * survivor selection: when every path's agreeing child beats every
//     disagreeing child (the common case at reliable positions) the survivors
//     are known after two warp reductions; otherwise a rank count over the
//     group's 2L candidates broadcast from shared memory, with an exact
//     (metric, index) pass only when the group holds tied metrics.
#include "args.cuh"
#include "scl_math.cuh"

namespace pc {

// Levels s..0 (s <= 2) in registers from source level s+1 at `src` (op at
// level s is g when `g`, with partial-sum bits `bits`; f below).  Stores the
// levels into the own slot (they are read again by later g steps and clones)
// and returns the level-0 soft value without reloading it.
template <bool FEX>
__device__ __forceinline__ float tail_from(float *own, const float *src, int s, uint32_t g, uint32_t bits)
{
    float l1a, l1b;
    if (s == 2) {
        const float4 A = *reinterpret_cast<const float4 *>(src);
        const float4 B = *reinterpret_cast<const float4 *>(src + 4);
        float4 o;
        if (g) {
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
        *reinterpret_cast<float4 *>(own + 4) = o;
        l1a = scl_f<FEX>(o.x, o.z);
        l1b = scl_f<FEX>(o.y, o.w);
    } else if (s == 1) {
        const float4 v = *reinterpret_cast<const float4 *>(src);
        l1a = g ? scl_g(v.x, v.z, bits & 1u) : scl_f<FEX>(v.x, v.z);
        l1b = g ? scl_g(v.y, v.w, (bits >> 1) & 1u) : scl_f<FEX>(v.y, v.w);
    } else {
        const float2 v = *reinterpret_cast<const float2 *>(src);
        const float lam = g ? scl_g(v.x, v.y, bits & 1u) : scl_f<FEX>(v.x, v.y);
        own[1] = lam;
        return lam;
    }
    *reinterpret_cast<float2 *>(own + 2) = make_float2(l1a, l1b);
    const float lam = scl_f<FEX>(l1a, l1b);
    own[1] = lam;
    return lam;
}

template <int L, bool FEX, int NV>
__global__ void __launch_bounds__(128) k_scl(const SclArgs a)
{
    constexpr int F = 32 / L;
    constexpr bool CH_SMEM = L >= 16;
    constexpr uint32_t FULL = 0xffffffffu;
    extern __shared__ __align__(16) uint32_t smw[];
    const int N = a.code.N, n = a.code.n, tp = a.tp, ss = a.ss, psw = a.psw, uhs = a.uhs;
    const int NW = (N + 31) >> 5;
    const int K = a.code.k, KW = (K + 31) >> 5;
    uint32_t *frz = smw;      // CTA-shared frozen mask
    uint32_t *dam = smw + NW; // CTA-shared decision-aided mask
    const int lane = threadIdx.x & 31;
    uint32_t *wbase = smw + a.table_words + (size_t)(threadIdx.x >> 5) * a.warp_words;
    float *llr = reinterpret_cast<float *>(wbase);
    uint32_t *ps = wbase + 32 * ss;
    uint32_t *uh = ps + 32 * psw;
    float *cand = reinterpret_cast<float *>(uh + 32 * uhs);
    float *chs = cand + 64;
    for (int w = threadIdx.x; w < NW; w += blockDim.x) {
        frz[w] = a.code.frozen_bits[w];
        dam[w] = a.code.da_bits != nullptr ? a.code.da_bits[w] : 0u;
    }
    __syncthreads();

    const int grp = lane / L, gbase = grp * L, pl = lane - gbase;
    const uint32_t gmask_lo = (L == 32) ? FULL : ((1u << L) - 1u);
    const int total = a.count != nullptr ? *a.count : a.B;
    float *own = llr + lane * ss;
    uint32_t *urow = uh + lane * uhs;
    uint32_t *prow = ps + lane * psw;
    float *cg = cand + grp * 2 * L;

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
        if (CH_SMEM) {
            float *mine = chs + grp * N;
            const float *g = a.llr + (size_t)frame * N;
            if (N >= 4) { // rows of N >= 4 floats are 16-byte aligned
                for (int t = 4 * pl; t < N; t += 4 * L)
                    *reinterpret_cast<float4 *>(mine + t) = __ldg(reinterpret_cast<const float4 *>(g + t));
            } else {
                for (int t = pl; t < N; t += L)
                    mine[t] = __ldg(g + t);
            }
            ch = mine;
            __syncwarp();
        } else {
            ch = a.llr + (size_t)frame * N;
        }

        uint64_t lanepat = 0; // the lane index in every 5-bit pointer field
        for (int s = 0; s < 12; ++s)
            lanepat = set_slot(lanepat, s, lane);
        uint64_t pll = lanepat, ppp = lanepat; // slot pointers: LLR levels, partial-sum levels
        int P = grp_live ? 1 : 0;
        int ji = 0; // index of the next non-frozen position (decisions are stored per info index)
        float metric = 0.0f;

        for (int i = 0; i < N; ++i) {
            const bool act = pl < P;
            // ---- descent: levels min(start, tp) .. 0 ----
            float lam = 0.0f;
            if (act) {
                const int start = (i == 0) ? n - 1 : __ffs(i) - 1;
                const int s0 = start < tp ? start : tp;
                const int w0 = 1 << s0;
                const uint32_t g0 = (i >> s0) & 1;
                float *dst = own + w0;
                const uint32_t *pw0 = ps + slot_of(ppp, s0) * psw + ps_off(s0);
                int top = s0; // highest level written to the own slot, -1 once lam is known
                if (s0 + 1 <= tp) {
                    // the only level read through a slot pointer; everything below is own
                    const float *src = llr + slot_of(pll, s0 + 1) * ss + 2 * w0;
                    if (s0 >= 3) {
                        if (g0)
                            level_from<FEX, true>(dst, src, w0, pw0);
                        else
                            level_from<FEX, false>(dst, src, w0, pw0);
                    } else {
                        lam = tail_from<FEX>(own, src, s0, g0, g0 ? pw0[0] : 0u);
                        top = -1;
                    }
                } else if (NV == 0) {
                    // level n-1 straight from the channel
                    if (w0 >= 4) {
                        if (g0)
                            level_from<FEX, true>(dst, ch, w0, pw0);
                        else
                            level_from<FEX, false>(dst, ch, w0, pw0);
                    } else {
                        for (int t = 0; t < w0; ++t)
                            dst[t] = g0 ? scl_g(ch[t], ch[w0 + t], bitw(pw0, t)) : scl_f<FEX>(ch[t], ch[w0 + t]);
                    }
                } else if (w0 >= 4) {
                    if constexpr (NV > 0) {
                        const uint32_t *psp[NV];
                        uint32_t gm = 0;
#pragma unroll
                        for (int d = 0; d < NV; ++d) {
                            const int r = n - NV + d;
                            psp[d] = ps + slot_of(ppp, r) * psw + ps_off(r);
                            gm |= ((uint32_t)(i >> r) & 1u) << d;
                        }
                        for (int t = 0; t < w0; t += 4) {
                            const float4 A = virt_top4<NV, FEX>(ch, n, t, psp, gm);
                            const float4 B = virt_top4<NV, FEX>(ch, n, t + w0, psp, gm);
                            *reinterpret_cast<float4 *>(dst + t) = g0 ? g4(A, B, pw0[t >> 5] >> (t & 31)) : f4(A, B, FEX);
                        }
                    }
                } else {
                    if constexpr (NV > 0) {
                        const uint32_t *psp[NV];
                        uint32_t gm = 0;
#pragma unroll
                        for (int d = 0; d < NV; ++d) {
                            const int r = n - NV + d;
                            psp[d] = ps + slot_of(ppp, r) * psw + ps_off(r);
                            gm |= ((uint32_t)(i >> r) & 1u) << d;
                        }
                        for (int t = 0; t < w0; ++t) {
                            const float A = virt_top<NV, FEX>(ch, n, t, psp, gm);
                            const float B = virt_top<NV, FEX>(ch, n, t + w0, psp, gm);
                            dst[t] = g0 ? scl_g(A, B, bitw(pw0, t)) : scl_f<FEX>(A, B);
                        }
                    }
                }
                if (top >= 3) {
                    for (int s = top - 1; s >= 3; --s)
                        level_from<FEX, false>(own + (1 << s), own + (2 << s), 1 << s, nullptr);
                    lam = tail_from<FEX>(own, own + 8, 2, 0u, 0u);
                } else if (top >= 0) { // first level came from the channel / virtual levels of a tiny code
                    for (int s = top - 1; s >= 0; --s)
                        level_from<FEX, false>(own + (1 << s), own + (2 << s), 1 << s, nullptr);
                    lam = own[1];
                }
                const uint64_t low = (5 * (s0 + 1) >= 64) ? ~0ull : ((1ull << (5 * (s0 + 1))) - 1ull);
                pll = (pll & ~low) | (lanepat & low); // levels 0..s0 now live in the own slot
            }
            __syncwarp();
            const uint32_t fz = (frz[i >> 5] >> (i & 31)) & 1u;
            const uint32_t dz = (dam[i >> 5] >> (i & 31)) & 1u;
            float inc0, inc1;
            metric_incs(lam, a.metric_exact, inc0, inc1);
            uint32_t u = 0;
            int src = lane;
            if (fz | dz) {
                u = (dz && lam < 0.0f) ? 1u : 0u;
                if (act)
                    metric += u ? inc1 : inc0;
            } else {
                // ---- branch: 2L candidates, keep the L best by (metric, candidate index) ----
                const float c0 = act ? metric + inc0 : INFINITY;
                const float c1 = act ? metric + inc1 : INFINITY;
                float gmax = fminf(c0, c1), bmin = fmaxf(c0, c1);
#pragma unroll
                for (int off = 1; off < L; off <<= 1) {
                    gmax = fmaxf(gmax, __shfl_xor_sync(FULL, gmax, off));
                    bmin = fminf(bmin, __shfl_xor_sync(FULL, bmin, off));
                }
                if (__all_sync(FULL, !grp_live || (P == L && gmax < bmin))) {
                    // every agreeing child beats every disagreeing child: the survivors
                    // are the agreeing children, no slot moves, no clones
                    const bool z = c0 < c1;
                    u = z ? 0u : 1u;
                    if (act)
                        metric = z ? c0 : c1;
                } else {
                    bool k0 = act, k1 = act;
                    if (__any_sync(FULL, 2 * P > L)) {
                        cg[pl] = c0;
                        cg[L + pl] = c1;
                        __syncwarp();
                        int lt0 = 0, lt1 = 0;
                        if constexpr (2 * L >= 4) {
#pragma unroll
                            for (int j = 0; j < 2 * L; j += 4) {
                                const float4 v = *reinterpret_cast<const float4 *>(cg + j);
                                lt0 += (v.x < c0) + (v.y < c0) + (v.z < c0) + (v.w < c0);
                                lt1 += (v.x < c1) + (v.y < c1) + (v.z < c1) + (v.w < c1);
                            }
                        } else {
                            lt0 = (cg[0] < c0) + (cg[1] < c0);
                            lt1 = (cg[0] < c1) + (cg[1] < c1);
                        }
                        // no ties among the 2P finite candidates <=> their strict ranks sum to fc(fc-1)/2
                        int sum = (act ? lt0 + lt1 : 0);
#pragma unroll
                        for (int off = 1; off < L; off <<= 1)
                            sum += __shfl_xor_sync(FULL, sum, off);
                        const bool tie = sum != P * (2 * P - 1);
                        if (__any_sync(FULL, tie)) {
                            lt0 = 0;
                            lt1 = 0;
                            for (int j = 0; j < 2 * L; ++j) {
                                const float v = cg[j];
                                lt0 += (v < c0) || (v == c0 && j < pl);
                                lt1 += (v < c1) || (v == c1 && j < L + pl);
                            }
                        }
                        k0 = act && lt0 < L;
                        k1 = act && lt1 < L;
                        __syncwarp();
                    }
                    const uint32_t freeM = (__ballot_sync(FULL, act && !k0 && !k1) >> gbase) & gmask_lo;
                    const uint32_t dupM = (__ballot_sync(FULL, act && k0 && k1) >> gbase) & gmask_lo;
                    const int nf = __popc(freeM), nd = __popc(dupM);
                    const bool surv = act && (k0 || k1);
                    if (surv) {
                        u = k0 ? 0u : 1u;
                        metric = k0 ? c0 : c1;
                    } else {
                        const int r = act ? __popc(freeM & ((1u << pl) - 1u)) : nf + (pl - P);
                        if (r < nd) {
                            uint32_t m = dupM; // the r-th set bit of dupM is the parent this slot clones
                            for (int z = 0; z < r; ++z)
                                m &= m - 1u;
                            src = gbase + __ffs(m) - 1;
                        }
                    }
                    const float pc1 = __shfl_sync(FULL, c1, src);
                    const uint32_t pl_lo = __shfl_sync(FULL, (uint32_t)pll, src);
                    const uint32_t pl_hi = __shfl_sync(FULL, (uint32_t)(pll >> 32), src);
                    const uint32_t pp_lo = __shfl_sync(FULL, (uint32_t)ppp, src);
                    const uint32_t pp_hi = __shfl_sync(FULL, (uint32_t)(ppp >> 32), src);
                    if (src != lane) {
                        u = 1u;
                        metric = pc1;
                        pll = ((uint64_t)pl_hi << 32) | pl_lo;
                        ppp = ((uint64_t)pp_hi << 32) | pp_lo;
                        const uint32_t *from = uh + src * uhs;
                        for (int w = 0; w <= (ji >> 5); ++w)
                            urow[w] = from[w];
                    }
                    P = P == 0 ? 0 : P - nf + nd;
                    __syncwarp();
                }
            }
            if (pl < P) {
                // record the decision (info positions only: frozen bits are 0),
                // then fold it into the partial sums
                if (!fz) {
                    const uint32_t bm = 1u << (ji & 31);
                    urow[ji >> 5] = u ? (urow[ji >> 5] | bm) : (urow[ji >> 5] & ~bm);
                }
                const int S = __ffs(~i) - 1; // trailing ones of i
                if (S < n) {
                    uint32_t F5 = u;
                    const int lo = S < 5 ? S : 5;
                    for (int s = 0; s < lo; ++s) {
                        const int len = 1 << s;
                        const uint32_t pv = ps[slot_of(ppp, s) * psw + s];
                        F5 = ((pv ^ F5) & ((1u << len) - 1u)) | (F5 << len);
                    }
                    uint32_t *dst = prow + ps_off(S);
                    if (S <= 5) {
                        dst[0] = F5;
                    } else {
                        const int words = 1 << (S - 5);
                        for (int w = 0; w < words; ++w) {
                            uint32_t v = F5;
                            for (int s = 5; s < S; ++s)
                                if (((w >> (s - 5)) & 1) == 0)
                                    v ^= ps[slot_of(ppp, s) * psw + ps_off(s) + (w & ((1 << (s - 5)) - 1))];
                            dst[w] = v;
                        }
                    }
                    ppp = set_slot(ppp, S, lane);
                }
            }
            ji += fz ? 0 : 1;
            __syncwarp();
        }

        // ---- winner: least (metric, slot) among CRC-passing paths (scl.py:177-191) ----
        const bool act = pl < P;
        bool ok = false;
        if (act && a.code.crc_width > 0) {
            uint32_t syn = 0;
            for (int w = 0; w < KW; ++w) {
                uint32_t v = urow[w];
                if (32 * w + 32 > K)
                    v &= (1u << (K & 31)) - 1u;
                while (v) {
                    const int b = __ffs(v) - 1;
                    v &= v - 1u;
                    syn ^= __ldg(a.code.crc_cols + __ldg(a.code.info_pos + 32 * w + b));
                }
            }
            ok = syn == a.code.crc_offset;
        }
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
        if (grp_live) {
            const uint32_t *row = uh + (gbase + who) * uhs;
            if (a.u_bits != nullptr)
                for (int w = pl; w < NW; w += L) {
                    // scatter the info bits back to block positions (frozen = 0)
                    int rank = 32 * w;
                    for (int z = 0; z < w; ++z)
                        rank -= __popc(frz[z]);
                    uint32_t v = 0;
                    for (int b = 0; b < 32 && 32 * w + b < N; ++b)
                        if (!((frz[w] >> b) & 1u))
                            v |= bitw(row, rank++) << b;
                    a.u_bits[(size_t)frame * NW + w] = v;
                }
            if (a.payload != nullptr) {
                const int MW = (a.code.m + 31) >> 5;
                for (int w = pl; w < MW; w += L) {
                    uint32_t v = row[w]; // payload = the first m info bits
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

int scl_prepare(SclArgs &a, int nv_req)
{
    const int n = a.code.n;
    int nv = nv_req;
    if (nv < 0)
        nv = 0;
    if (nv > n - 2)
        nv = n - 2 > 0 ? n - 2 : 0; // keep at least levels 0..1 stored (float4 needs tp >= 2 anyway)
    if (nv > 4)
        nv = 4;
    // v2 is the fallback kernel (N < 16, or the kernel = 1 knob): compiled for NV in {0, 3} only
    nv = nv >= 3 ? 3 : 0;
    a.nv = nv;
    a.tp = n - 1 - nv;
    a.ss = (1 << (a.tp + 1)) + 4;
    a.psw = ps_off(n) | 1; // words for levels 0..n-1, odd stride
    const int nw = (a.code.N + 31) >> 5;
    (void)nw;
    a.uhs = ((a.code.k + 31) >> 5) | 1; // decisions at the k non-frozen positions
    a.table_words = (2 * nw + 3) & ~3;
    return PC_OK;
}

template <int L, bool FEX, int NV>
static int launch_scl_t(SclArgs a, int wpc, int max_warps, cudaStream_t s)
{
    auto kern = k_scl<L, FEX, NV>;
    constexpr int F = 32 / L;
    const int ch_words = (L >= 16) ? F * a.code.N : 0;
    a.warp_words = 32 * (a.ss + a.psw + a.uhs) + 64 + ch_words;
    a.warp_words = (a.warp_words + 3) & ~3;
    const size_t per_warp = (size_t)a.warp_words * 4;
    const size_t table = (size_t)a.table_words * 4;
    const size_t smem_cap = 227 * 1024;
    if (table + per_warp > smem_cap)
        return PC_ERR_UNSUPPORTED;
    while (wpc > 1 && table + (size_t)wpc * per_warp > smem_cap)
        --wpc;
    const size_t smem = table + (size_t)wpc * per_warp;
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
