// sc1.cu -- K3 for list size 1 (successive cancellation, reference sim.py:152-153:
// SC is scl_decode with L = 1): G frames per warp, 32/G lanes per frame (sm_100a).
//
// K3 v3 (scl3.cuh) maps 32 / L frames onto a warp, one lane per path, so at
// L = 1 every lane walks a whole frame alone: the upper tree levels (2^s
// elements each) run serially per lane, the virtual top levels re-read 32
// channel rows through L1/L2 per warp, and one frame takes ~0.9 ms at
// N = 2048.  Here a group of GL = 32/G lanes shares one frame:
//   * every upper level (5 .. n-1) is stored once per frame in shared memory
//     and computed element-parallel by the group (lane t of the group:
//     elements t, t + GL, ...), f or g with the stored partial sums; the
//     channel row is read (coalesced, from global memory) only for level n-1;
//   * each block of 32 leaves runs on the group's first lane from registers
//     with the same leaf code as K3 v3 (levels 4..0, their partial sums in one
//     word, the fp32 metric and the L = 1 decision rule c1 < c0 of the
//     (metric, index) order, _kernels.py:247-311), so decisions, metric and
//     CRC flag are bit-identical to K3 v3 at L = 1 (tools/sc1_ab.py,
//     tests/test_gpu_scl.py);
//   * the block's codeword is folded into the stored partial sums
//     element-parallel;
//   * the code tables (CRC syndrome columns, frozen and decision-aided words)
//     are staged once per CTA in shared memory, so a leaf's column read is not
//     a global-memory round trip on the decision chain.
// G = 1 is the latency form (one frame per warp, small batches); G = 8 or 4 the
// throughput form.  Shared memory per frame: levels 5..n-1 (N - 32 floats),
// partial sums N/32 words, decisions N/32 words.
#include "args.cuh"
#include "scl_math.cuh"

namespace pc {

namespace sc1 {
constexpr int T = 5; // leaf blocks of 32
__host__ __device__ constexpr int lvl(int s) { return (1 << s) - 32; }      // level s >= 5, floats
__host__ __device__ constexpr int pso(int s) { return (1 << (s - 5)) - 1; } // partial sums of level s >= 5, words
// Stored LLR levels 5..TP = min(n - 1, 8); the NV = n - 1 - TP levels above are
// recomputed from the channel (scl_math.cuh::virt_top) when the descent
// crosses them (each of levels 9..n-1 is visited 2^(n-1-s) times per frame), so
// a frame needs 2.5 KB of shared memory at N = 2048 instead of 8.5 KB.
#ifndef SC1_TOP
#define SC1_TOP 8
#endif
__host__ __device__ constexpr int top_level(int n) { return n - 1 < SC1_TOP ? n - 1 : SC1_TOP; }
__host__ __device__ inline int frame_words(int N, int n) // levels, partial sums, decisions, leaf LLRs, increments
{
    // a stride of 4 (mod 32) words: the G frames of a warp (32/G lanes each,
    // consecutive elements) fall in distinct banks (with a multiple of 32 they
    // all hit the same ones: ncu measured 84% of the shared wavefronts as conflicts)
    return (((2 << top_level(n)) - 32 + 2 * (N / 32) + 96 + 31) & ~31) + 4;
}
// CTA tables: 32 zero words (the CRC columns of a code without a CRC; the
// columns themselves are read through L1, in the latency form one per lane,
// issued before the block's descent), frozen and decision-aided words
template <int G>
__host__ __device__ inline int table_words(int N) { return 32 + 2 * (N / 32); }
} // namespace sc1

// Shared words of one warp: its G frames, plus (G = 1) the frame's deferred metric
// terms and its channel row (the upper levels re-read it; from global memory
// every read is an L2 round trip on the single warp's critical path).
template <int G>
__host__ __device__ inline int sc1_frame_words(int N, int n)
{
    return G * sc1::frame_words(N, n) + (G == 1 ? 3 * N + 4 + ((N / 32 + 3) & ~3) : 0);
}

// One block of 32 leaves from its level-5 LLRs x (K3 v3's leaf code at L = 1):
// decisions bu, the fp32 metric, the CRC syndrome and the block codeword betaT.
// SPEC = false: the exact rule at every leaf (decision c1 < c0 of the metric
// sums, _kernels.py:247-311), one dependent chain through MUFU and the metric.
// SPEC = true: the decision chain takes u = (lam < 0) at info leaves (what the
// rule decides unless metric + inc0 and metric + inc1 round to the same fp32
// value), keeping the MUFU work and the metric off it; a second, unrolled pass
// then evaluates the exact rule from the stored leaf LLRs and returns false if
// any decision would differ (the caller replays the block with SPEC = false),
// so the result is bit-identical either way.
// One leaf j of a 32-leaf block (K3 v3's leaf code at L = 1): the leaf LLR from
// the register levels, the decision and the partial-sum fold.  SPEC: the
// decision u = (lam < 0) at info leaves and the LLR kept in lamS[j] for the
// metric pass; else the exact rule (decision c1 < c0 of the fp32 metric sums,
// _kernels.py:247-311) with the metric update.
template <bool FEX, bool SPEC>
__device__ __forceinline__ void leaf_step(int j, const float (&x)[32], float (&l4)[16], float (&l3)[8], float (&l2)[4],
                                          float (&l1)[2], uint32_t &psr, uint32_t fzw, uint32_t daw, uint32_t col,
                                          int metric_exact, float *lamS, float &metric, uint32_t &syn, uint32_t &bu,
                                          uint32_t &betaT)
{
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
    uint32_t u;
    if constexpr (SPEC) {
        // the decision the metric rule takes unless c0 and c1 round alike
        u = (!fz && lam < 0.0f) ? 1u : 0u;
        lamS[j] = lam;
    } else {
        float inc0, inc1;
        metric_incs(lam, metric_exact, inc0, inc1);
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
    }
    if (!fz && u)
        syn ^= col;
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

// The decision chain of one block of 32 leaves from its level-5 LLRs x:
// decisions bu, the CRC syndrome and the block codeword betaT.
// SPEC = true: u = (lam < 0) at info leaves (what the exact rule decides unless
// metric + inc0 and metric + inc1 round to the same fp32 value), the leaf LLRs
// kept in lamS for the metric pass; unrolled, so every branch on j and every
// partial-sum bit position is resolved at compile time.
// SPEC = false: the exact rule with the metric at every leaf (the replay when
// the metric pass rejects a speculative decision; one copy of the leaf code).
template <bool FEX, bool SPEC>
__device__ __forceinline__ void leaf_chain(const float (&x)[32], uint32_t fzw, uint32_t daw, const uint32_t *cols,
                                           int metric_exact, float *lamS, float &metric, uint32_t &syn, uint32_t &bu,
                                           uint32_t &betaT)
{
    float l4[16], l3[8], l2[4], l1[2];
    uint32_t psr = 0;
    bu = 0;
    if constexpr (SPEC) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            leaf_step<FEX, true>(j, x, l4, l3, l2, l1, psr, fzw, daw, cols[j], metric_exact, lamS, metric, syn, bu,
                                 betaT);
    } else {
#pragma unroll 1
        for (int j = 0; j < 32; ++j)
            leaf_step<FEX, false>(j, x, l4, l3, l2, l1, psr, fzw, daw, cols[j], metric_exact, lamS, metric, syn, bu,
                                  betaT);
    }
}

// The exact rule over a block from precomputed increments inc[2j] (u = 0),
// inc[2j + 1] (u = 1): the metric in leaf order, and true if every
// speculative decision in bu is what the rule decides (bit-identical result).
__device__ __forceinline__ bool metric_pass(uint32_t fzw, uint32_t daw, uint32_t bu, const float *inc, float &metric)
{
    bool same = true;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        const float4 v = *reinterpret_cast<const float4 *>(inc + 2 * j);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int jj = j + h;
            const float inc0 = h ? v.z : v.x, inc1 = h ? v.w : v.y;
            const uint32_t fz = (fzw >> jj) & 1u, dz = (daw >> jj) & 1u, us = (bu >> jj) & 1u;
            if (fz | dz) {
                metric += us ? inc1 : inc0;
            } else {
                const float c0 = metric + inc0, c1 = metric + inc1;
                const uint32_t u = c1 < c0 ? 1u : 0u;
                same &= u == us;
                metric = u ? c1 : c0;
            }
        }
    }
    return same;
}

// The polar transform of a 32-bit word (bit i = position i): [a xor b, b]
// recursively, the same bit layout as the leaf code's block codeword.  An
// involution, so it also maps a codeword back to its decisions.
__device__ __forceinline__ uint32_t polar32(uint32_t v)
{
    v ^= (v >> 1) & 0x55555555u;
    v ^= (v >> 2) & 0x33333333u;
    v ^= (v >> 4) & 0x0F0F0F0Fu;
    v ^= (v >> 8) & 0x00FF00FFu;
    v ^= (v >> 16) & 0x0000FFFFu;
    return v;
}

// Leaf LLRs of a 32-leaf block for given decisions u (bit j = leaf j), one
// leaf per lane: the block's subtree breadth-first, level s holding element
// (lane & (2^s - 1)) of node (lane >> s); a node's two parent elements sit in
// lanes lane and lane ^ 2^s.  The g operations take the left sibling's
// codeword from the partial transforms T_s of u.  Same f / g on the same
// values as the leaf code, so the LLRs are bit-identical to it whenever u
// agrees with the decisions before each leaf.
template <bool FEX>
__device__ __forceinline__ float leaves32(float xl, uint32_t u, int lane)
{
    uint32_t T[5];
    T[0] = u;
    T[1] = T[0] ^ ((T[0] >> 1) & 0x55555555u);
    T[2] = T[1] ^ ((T[1] >> 2) & 0x33333333u);
    T[3] = T[2] ^ ((T[2] >> 4) & 0x0F0F0F0Fu);
    T[4] = T[3] ^ ((T[3] >> 8) & 0x00FF00FFu);
    float v = xl;
#pragma unroll
    for (int s = 4; s >= 0; --s) {
        const int h = 1 << s;
        const float p = __shfl_xor_sync(0xffffffffu, v, h);
        if (lane & h) // right child: g with the left sibling's codeword
            v = scl_g(p, v, (T[s] >> (lane & ~h)) & 1u);
        else
            v = scl_f<FEX>(v, p);
    }
    return v;
}

#ifndef SC1_CN
#define SC1_CN 1
#endif

// DEF: the default knobs compiled in (exact metric, CRC on, no decision-aided
// positions); the launcher picks it when the arguments match.
template <bool FEX, int G, int NV, bool DEF = false>
__global__ void __launch_bounds__(128) k_sc1(const SclArgs a)
{
    using namespace sc1;
    constexpr uint32_t FULL = 0xffffffffu;
    constexpr int GL = 32 / G; // lanes per frame
    extern __shared__ __align__(16) uint32_t smw[];
    // with virtual levels the launcher picked NV = n - SC1_TOP - 1: the code
    // length is a compile-time constant then (address arithmetic in immediates)
    const int n = (NV > 0 && SC1_CN) ? SC1_TOP + 1 + NV : a.code.n;
    const int N = 1 << n, NW = N >> 5;
    const int lane = threadIdx.x & 31, grp = lane / GL, pl = lane % GL;
    uint32_t *colS = smw;
    uint32_t *frzS = colS + 32;
    uint32_t *daS = frzS + NW;
    const bool use_crc = DEF ? true : a.code.crc_width > 0;
    const int mex = DEF ? 1 : a.metric_exact;
    for (int i = threadIdx.x; i < N; i += blockDim.x)
        if (i < 32)
            colS[i] = 0u;
    for (int i = threadIdx.x; i < NW; i += blockDim.x) {
        frzS[i] = a.code.frozen_bits[i];
        daS[i] = a.code.da_bits != nullptr ? a.code.da_bits[i] : 0u;
    }
    __syncthreads();
    const int tp = NV > 0 ? SC1_TOP : n - 1; // top stored level
    float *lv = reinterpret_cast<float *>(smw + table_words<G>(N) + (size_t)(threadIdx.x >> 5) * sc1_frame_words<G>(N, n) +
                                          grp * frame_words(N, n));
    uint32_t *ps = reinterpret_cast<uint32_t *>(lv + (2 << tp) - 32);
    uint32_t *ub = ps + NW;
    float *lam = reinterpret_cast<float *>(ub + NW); // 32 leaf LLRs of the current block
    float *inc = lam + 32;                            // their metric increments (u = 0, u = 1)
    // G = 1: the frame's deferred metric terms (chosen / other increment per leaf, confirm bits)
    float *incS = reinterpret_cast<float *>(smw) + table_words<G>(N) + (size_t)(threadIdx.x >> 5) * sc1_frame_words<G>(N, n) +
                  frame_words(N, n);
    float *incO = incS + N + 4;
    uint32_t *chk = reinterpret_cast<uint32_t *>(incO + N);
    float *chS = incO + N + ((NW + 3) & ~3); // G = 1: the channel row
    const int total = a.count != nullptr ? *a.count : a.B;
    const int nblk = N >> T;

    // work == nullptr: the launch holds a warp for every G frames (small batches),
    // so frames go by warp index and no counter has to be reset first
    const int static_base = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * G;
    for (int round = 0;; ++round) {
        int base = 0;
        if (a.work == nullptr) {
            base = round == 0 ? static_base : total;
        } else {
            if (lane == 0)
                base = atomicAdd(a.work, G);
            base = __shfl_sync(FULL, base, 0);
        }
        if (base >= total)
            break;
        const int qi = base + grp;
        const bool live = qi < total;
        const int frame = live ? (a.queue != nullptr ? a.queue[qi] : qi) : 0;
        const float *ch = a.llr + (size_t)frame * N;
        if constexpr (G == 1) {
            const float4 *g4p = reinterpret_cast<const float4 *>(ch);
            for (int t = lane; t < N / 4; t += 32)
                reinterpret_cast<float4 *>(chS)[t] = __ldg(g4p + t);
            __syncwarp();
            ch = chS;
        }
        float metric = 0.0f, m_blk = 0.0f; // m_blk, s_blk: metric and syndrome at the block's start
        uint32_t syn = 0u, s_blk = 0u;
        // G = 1: pass 0 decides every block by the fixpoint and defers the metric to
        // one chain over the frame's leaves; if that chain rejects a decision (or a
        // fixpoint did not settle), pass 1 decodes the frame again with the exact
        // per-block path.  G > 1: the per-block path only.
        for (int pass = (G == 1 ? 0 : 1); pass < 2; ++pass) {
        const bool fast = G == 1 && pass == 0;
        metric = m_blk = 0.0f;
        syn = s_blk = 0u;
        bool settled = true;
        for (int b = 0; b < nblk; ++b) {
            const int i0 = b << T;
            // (latency form: this lane's CRC column of the block, in flight during the descent)
            const uint32_t colv = G == 1 && use_crc ? __ldg(a.code.crc_cols + i0 + lane) : 0u;
            // ---- upper descent: levels start..5, element-parallel over the group ----
            const int start = (b == 0) ? n - 1 : T + __ffs(b) - 1;
            for (int s = start < tp ? start : tp; s >= T; --s) {
                const int w = 1 << s;
                float *dst = lv + lvl(s);
                const bool g = (i0 >> s) & 1;
                const uint32_t *pw = ps + pso(s);
                if constexpr (NV > 0) {
                    if (s == tp) { // (its source level tp + 1 is virtual)
                        // level tp from the virtual levels n-NV..n-1 (recomputed from the channel)
                        const uint32_t *psp[NV];
                        uint32_t gm = 0;
#pragma unroll
                        for (int d = 0; d < NV; ++d) {
                            psp[d] = ps + pso(n - NV + d);
                            gm |= ((uint32_t)(i0 >> (n - NV + d)) & 1u) << d;
                        }
                        for (int t = pl; t < w; t += GL) {
                            const float A = virt_top<NV, FEX>(ch, n, t, psp, gm);
                            const float B = virt_top<NV, FEX>(ch, n, t + w, psp, gm);
                            dst[t] = g ? scl_g(A, B, (pw[t >> 5] >> (t & 31)) & 1u) : scl_f<FEX>(A, B);
                        }
                        __syncwarp();
                        continue;
                    }
                }
                if (s + 1 == n) { // from the channel (global memory, coalesced)
                    for (int t = pl; t < w; t += GL) {
                        const float A = ch[t], B = ch[t + w];
                        dst[t] = g ? scl_g(A, B, (pw[t >> 5] >> (t & 31)) & 1u) : scl_f<FEX>(A, B);
                    }
                } else {
                    const float *src = lv + lvl(s + 1);
                    for (int t = pl; t < w; t += GL) {
                        const float A = src[t], B = src[t + w];
                        dst[t] = g ? scl_g(A, B, (pw[t >> 5] >> (t & 31)) & 1u) : scl_f<FEX>(A, B);
                    }
                }
                __syncwarp();
            }
            // ---- the block's 32 leaves on the group's first lane, registers only
            // (K3 v3's leaf code at L = 1) ----
            uint32_t betaT = 0, bu = 0;
            const uint32_t fzw = frzS[b], daw = DEF ? 0u : daS[b];
            if (fast) {
                // One frame per warp (latency form): the block's decisions as the fixpoint
                // of u = rule(lambda(u)), one leaf per lane.  lambda_j depends on u_0..u_j-1
                // only, so after round r the first r decisions are final and the fixpoint
                // (reached in <= 32 rounds, typically 1-3 from the hard-decision guess) is
                // the sequential decoder's.  The rule here is u = (lambda < 0) at info
                // leaves; the metric pass below checks it against the exact rule.
                const float xl = lv[lane];
                const uint32_t info = ~fzw;
                uint32_t u = polar32(__ballot_sync(FULL, xl < 0.0f)) & info;
                float laml = 0.0f;
                bool conv = false;
                for (int r = 0; r < 40; ++r) {
                    laml = leaves32<FEX>(xl, u, lane);
                    const uint32_t un = __ballot_sync(FULL, laml < 0.0f) & info;
                    if (un == u) {
                        conv = true;
                        break;
                    }
                    u = un;
                }
                settled &= conv;
                bu = u;
                betaT = polar32(u);
                syn ^= __reduce_xor_sync(FULL, ((u >> lane) & 1u) ? colv : 0u);
                // the leaf's increment for its decision, the other one, and whether the
                // exact rule must confirm the decision (info leaf decided 1: the rule keeps
                // u = 1 only if metric + inc1 < metric + inc0; a leaf decided 0 has
                // inc0 <= inc1 and stays 0)
                float i0v, i1v;
                metric_incs(laml, mex, i0v, i1v);
                const bool u1 = (u >> lane) & 1u;
                incS[i0 + lane] = u1 ? i1v : i0v;
                incO[i0 + lane] = u1 ? i0v : i1v;
                const uint32_t ck = __ballot_sync(FULL, u1 && !((daw >> lane) & 1u));
                if (lane == 0) {
                    chk[b] = ck;
                    ub[b] = bu;
                }
            } else {
            float x[32];
            if (pl == 0) { // the decision chain (speculative), leaf LLRs into lam[]
#pragma unroll
                for (int t = 0; t < 32; t += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(lv + t);
                    x[t] = v.x, x[t + 1] = v.y, x[t + 2] = v.z, x[t + 3] = v.w;
                }
                leaf_chain<FEX, true>(x, fzw, daw, use_crc ? a.code.crc_cols + i0 : colS, mex, lam, metric,
                                      syn, bu, betaT);
            }
            __syncwarp();
            // the metric increments of the 32 leaves, element-parallel over the group
            for (int j = pl; j < 32; j += GL) {
                float i0v, i1v;
                metric_incs(lam[j], mex, i0v, i1v);
                inc[2 * j] = i0v;
                inc[2 * j + 1] = i1v;
            }
            __syncwarp();
            if (pl == 0) {
                // the exact rule from the increments: the metric, and whether every
                // speculative decision stands
                if (!metric_pass(fzw, daw, bu, inc, metric)) {
                    // an info decision hinged on the metric's rounding: exact replay of the
                    // block from its start (metric and syndrome as they were)
                    metric = m_blk;
                    syn = s_blk;
                    leaf_chain<FEX, false>(x, fzw, daw, use_crc ? a.code.crc_cols + i0 : colS, mex, lam,
                                           metric, syn, bu, betaT);
                }
                m_blk = metric;
                s_blk = syn;
                ub[b] = bu;
            }
            }
            // ---- block end: fold the block codeword into the stored partial sums ----
            betaT = __shfl_sync(FULL, betaT, grp * GL);
            const int S = T + __ffs(~b) - 1; // level of the node this block completes
            if (S < n) {
                const int words = 1 << (S - T);
                for (int w = pl; w < words; w += GL) {
                    uint32_t v = betaT;
                    for (int s = T; s < S; ++s)
                        if (((w >> (s - T)) & 1) == 0)
                            v ^= ps[pso(s) + (w & ((1 << (s - T)) - 1))];
                    ps[pso(S) + w] = v;
                }
            }
            __syncwarp();
        }
        if (!fast)
            break;
        // the frame's metric: one fp32 chain over the leaves in order (the reference's
        // order of additions) on lane 0, writing the metric before each leaf over its
        // chosen increment; then every lane checks its leaves: a leaf the exact rule
        // must confirm keeps u = 1 only if (metric before) + inc1 < (metric before) + inc0
        if (lane == 0) {
            float m = 0.0f;
            for (int i = 0; i < N; i += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(incS + i);
                float4 pre;
                pre.x = m;
                m += v.x;
                pre.y = m;
                m += v.y;
                pre.z = m;
                m += v.z;
                pre.w = m;
                m += v.w;
                *reinterpret_cast<float4 *>(incS + i) = pre; // incS[i] := the metric before leaf i
            }
            metric = m;
            incS[N] = m; // (the metric after the last leaf)
        }
        __syncwarp();
        bool ok = settled;
        for (int i = lane; i < N; i += 32)
            if ((chk[i >> 5] >> (i & 31)) & 1u)
                ok &= incS[i + 1] < incS[i] + incO[i];
        ok = __all_sync(FULL, ok);
        if (ok)
            break;
        }
        // ---- outputs (the one path is the winner, scl.py:177-191) ----
        metric = __shfl_sync(FULL, metric, grp * GL);
        syn = __shfl_sync(FULL, syn, grp * GL);
        if (live) {
            if (a.u_bits != nullptr)
                for (int w = pl; w < NW; w += GL)
                    a.u_bits[(size_t)frame * NW + w] = ub[w];
            if (a.payload != nullptr) {
                const int m = a.code.m, MW = (m + 31) >> 5;
                for (int w = pl; w < MW; w += GL) {
                    uint32_t v = 0u;
                    for (int q = 0; q < 32 && 32 * w + q < m; ++q) {
                        const int p = __ldg(a.code.info_pos + 32 * w + q);
                        v |= ((ub[p >> 5] >> (p & 31)) & 1u) << q;
                    }
                    a.payload[(size_t)frame * MW + w] = v;
                }
            }
            if (pl == 0) {
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
        }
        __syncwarp();
    }
}

bool sc1_eligible(const SclArgs &a) { return a.code.n >= 6 && a.code.n <= 12; }

template <bool FEX, int G, int NV>
static int launch_sc1_t(const SclArgs &a, cudaStream_t s, long long *capacity = nullptr)
{
    auto kern = k_sc1<FEX, G, NV>;
    if constexpr (!FEX && NV > 0 && SC1_CN)
        if (a.metric_exact && a.code.crc_width > 0 && a.code.da_bits == nullptr)
            kern = k_sc1<FEX, G, NV, true>;
    const int N = a.code.N, n = a.code.n;
    auto bytes = [&](int w) { return ((size_t)sc1::table_words<G>(N) + (size_t)w * sc1_frame_words<G>(N, n)) * 4; };
    if (bytes(1) > 227 * 1024)
        return PC_ERR_UNSUPPORTED;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
        return PC_ERR_CUDA;
    // warps per CTA: the most frames resident per SM (each CTA carries the tables
    // once; registers allow 16 warps per SM), fewer warps on a tie
    // (G = 1, the latency form: four warps, so the CTA stages the tables fast)
    int wpc = 1, best = 0;
    for (int w = G == 1 ? 4 : 1; w <= 4; ++w) {
        int per_sm = 0;
        if (bytes(w) > 227 * 1024 ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * w, bytes(w)) != cudaSuccess)
            break;
        if (per_sm * w * G > best) {
            best = per_sm * w * G;
            wpc = w;
        }
    }
    cudaGetLastError();
    if (best == 0)
        return PC_ERR_UNSUPPORTED;
    const size_t smem = bytes(wpc);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (capacity != nullptr) { // (a query: frames resident at once, no launch)
        *capacity = (long long)sms * best;
        return PC_OK;
    }
    long long grid = (long long)sms * (best / (wpc * G));
    const long long need = ((long long)a.B + (long long)wpc * G - 1) / ((long long)wpc * G);
    SclArgs b = a;
    if (grid >= need && a.count == nullptr) {
        grid = need; // one warp per G frames: static assignment, no counter
        b.work = nullptr;
    } else if (cudaMemsetAsync(a.work, 0, sizeof(int32_t), s) != cudaSuccess) {
        return PC_ERR_CUDA;
    }
    kern<<<(int)grid, 32 * wpc, smem, s>>>(b);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

template <bool FEX, int G>
static int launch_sc1_g(const SclArgs &a, cudaStream_t s, long long *capacity = nullptr)
{
    switch (a.code.n > SC1_TOP + 1 ? a.code.n - SC1_TOP - 1 : 0) { // NV: virtual levels above the top stored level
    case 0: return launch_sc1_t<FEX, G, 0>(a, s, capacity);
    case 1: return launch_sc1_t<FEX, G, 1>(a, s, capacity);
    case 2: return launch_sc1_t<FEX, G, 2>(a, s, capacity);
    case 3: return launch_sc1_t<FEX, G, 3>(a, s, capacity);
    case 4: return launch_sc1_t<FEX, G, 4>(a, s, capacity);
    }
    return PC_ERR_UNSUPPORTED;
}

template <bool FEX>
static int launch_sc1_f(const SclArgs &a, cudaStream_t s, int sms)
{
    // G = 1 (latency form, one frame per warp) while the batch fits one frame per
    // resident warp; else 8 frames per warp when the batch then fits one wave of
    // resident frames, 4 when it does not (measured at N = 2048: 4 frames per warp
    // run each wave faster, 8 hold more frames at once: 10^4 frames 16.1 vs 12.9
    // Mframes/s, 32768 frames 14.7 vs 19.1)
    if (a.B <= sms * 8)
        return launch_sc1_g<FEX, 1>(a, s);
    long long cap8 = 0;
    if (launch_sc1_g<FEX, 8>(a, s, &cap8) == PC_OK && a.B <= cap8)
        return launch_sc1_g<FEX, 8>(a, s);
    return launch_sc1_g<FEX, 4>(a, s);
}

int launch_sc1(const SclArgs &a, cudaStream_t s)
{
    if (a.B == 0)
        return PC_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return a.f_exact ? launch_sc1_f<true>(a, s, sms) : launch_sc1_f<false>(a, s, sms);
}

} // namespace pc
