// scl_math.cuh -- SCL node arithmetic shared by K3 v2 (scl.cu) and v3 (scl3.cu).
// Restates the primitives of _kernels.py:40-90 in fp32 (reference
// /root/reference/pkg/src/polarsim/_kernels.py).
#pragma once
#include "common.cuh"

namespace pc {

// _kernels.py:40-48.  When either input is zero the magnitude is zero; the
// sign bit of that zero is irrelevant downstream (f, g, the metric and the
// hard decision treat -0 and +0 alike).
__device__ __forceinline__ float f_minsum(float a, float b)
{
    const float mag = fminf(fabsf(a), fabsf(b));
    return __uint_as_float(__float_as_uint(mag) | ((__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u));
}

// _kernels.py:51-65 computes f = logaddexp(0, a+b) - logaddexp(a, b) in fp64.
// The same difference in fp32 loses the result to cancellation whenever |f|
// is small against |a| + |b| (absolute error ~ulp(|a| + |b|), e.g. f(20, 1e-3)
// to 0.2%; deep f chains of high-rate codes at N = 4096 then decide other
// paths).  Two cancellation-free forms of the same function instead, with
// x = max(|a|, |b|), y = min(|a|, |b|), f = sign(a) sign(b) |f|:
//   x < 4:  |f| = 2 atanh(tanh(x/2) tanh(y/2))     (product < tanh(2)^2 = 0.93)
//   x >= 4: |f| = y - log1p(z),  z = (e^(y-x) - e^-(x+y)) / (1 + e^-(x+y)) <= 0.04 y / (1 - 0.04)
// (the second is log((1 + e^(x+y)) / (e^x + e^y)) rearranged: no difference
// of large terms).  Relative error ~1e-7 in both ranges.
__device__ __forceinline__ float f_boxplus(float a, float b)
{
    const float ax = fabsf(a), bx = fabsf(b);
    const float x = fmaxf(ax, bx), y = fminf(ax, bx);
    float m;
    if (x < 4.0f) {
        m = 2.0f * atanhf(tanhf(0.5f * x) * tanhf(0.5f * y));
    } else {
        const float e = expf(-(x + y));
        m = y - log1pf((expf(y - x) - e) / (1.0f + e));
    }
    return __uint_as_float(__float_as_uint(m) | ((__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u));
}

template <bool FEX>
__device__ __forceinline__ float scl_f(float a, float b)
{
    return FEX ? f_boxplus(a, b) : f_minsum(a, b);
}

// _kernels.py:68-73: b + (1 - 2u) a  (b - a == b + (-a) exactly in IEEE)
__device__ __forceinline__ float scl_g(float a, float b, uint32_t u)
{
    return b + __uint_as_float(__float_as_uint(a) ^ (u << 31));
}

// Metric increments for both decisions at soft value lam (_kernels.py:76-90).
__device__ __forceinline__ void metric_incs(float lam, bool exact, float &inc0, float &inc1)
{
    if (exact) {
        // sp = log1p(exp(-|lam|)) on the MUFU pipe: ex2 then lg2(1 + e); for
        // e < 2^-10 the two-term series e (1 - e/2) is more accurate than lg2
        // of a value that close to 1.  Absolute error < 2e-7, below the fp32
        // rounding of the metrics it is added to.
        const float y = fabsf(lam);
        const float e = ex2_approx(-y * PC_LOG2E);
        const float sp = e < 0.0009765625f ? e * (1.0f - 0.5f * e) : PC_LN2 * lg2_approx(1.0f + e);
        const float agree = sp, disagree = y + sp;
        // x = lam for u = 0: x > 0 -> sp(x); x <= 0 -> -x + sp(-x)
        inc0 = lam > 0.0f ? agree : disagree;
        inc1 = lam < 0.0f ? agree : disagree;
    } else {
        inc0 = lam < 0.0f ? -lam : 0.0f;
        inc1 = lam > 0.0f ? lam : 0.0f;
    }
}

// word offset of partial-sum level s: levels <= 5 take one word, level s > 5 takes 2^(s-5)
__host__ __device__ __forceinline__ int ps_off(int s) { return s <= 5 ? s : (1 << (s - 5)) + 4; }

__device__ __forceinline__ int slot_of(uint64_t ptrs, int s) { return (int)((ptrs >> (5 * s)) & 31u); }
__device__ __forceinline__ uint64_t set_slot(uint64_t ptrs, int s, int v)
{
    return (ptrs & ~(31ull << (5 * s))) | ((uint64_t)v << (5 * s));
}

__device__ __forceinline__ uint32_t bitw(const uint32_t *p, int x) { return (p[x >> 5] >> (x & 31)) & 1u; }

// Element t of the highest virtual level s = n - NV, recomputed bottom-up from
// the 2^NV channel leaves t + j 2^s.  psp[d] = partial-sum words of level s+d,
// bit d of gmask = the op at level s+d is g.
template <int NV, bool FEX>
__device__ __forceinline__ float virt_top(const float *ch, int n, int t, const uint32_t *const *psp, uint32_t gmask)
{
    constexpr int CNT = 1 << (NV - 1);
    const int s = n - NV;
    const int half = 1 << (n - 1);
    float v[CNT];
#pragma unroll
    for (int j = 0; j < CNT; ++j) {
        const int x = t + (j << s);
        const float A = ch[x], B = ch[x + half];
        v[j] = ((gmask >> (NV - 1)) & 1u) ? scl_g(A, B, bitw(psp[NV - 1], x)) : scl_f<FEX>(A, B);
    }
#pragma unroll
    for (int d = NV - 2; d >= 0; --d) {
        const int c = 1 << d;
#pragma unroll
        for (int j = 0; j < c; ++j) {
            const int x = t + (j << s);
            v[j] = ((gmask >> d) & 1u) ? scl_g(v[j], v[j + c], bitw(psp[d], x)) : scl_f<FEX>(v[j], v[j + c]);
        }
    }
    return v[0];
}

__device__ __forceinline__ float4 f4(const float4 A, const float4 B, bool fex)
{
    float4 o;
    if (fex) {
        o.x = f_boxplus(A.x, B.x);
        o.y = f_boxplus(A.y, B.y);
        o.z = f_boxplus(A.z, B.z);
        o.w = f_boxplus(A.w, B.w);
    } else {
        o.x = f_minsum(A.x, B.x);
        o.y = f_minsum(A.y, B.y);
        o.z = f_minsum(A.z, B.z);
        o.w = f_minsum(A.w, B.w);
    }
    return o;
}

__device__ __forceinline__ float4 g4(const float4 A, const float4 B, uint32_t bits)
{
    return make_float4(scl_g(A.x, B.x, bits & 1u), scl_g(A.y, B.y, (bits >> 1) & 1u), scl_g(A.z, B.z, (bits >> 2) & 1u),
                       scl_g(A.w, B.w, (bits >> 3) & 1u));
}

// Vector form of virt_top: elements t..t+3 (t % 4 == 0) of the highest
// virtual level; one partial-sum word serves all four elements.
template <int NV, bool FEX>
__device__ __forceinline__ float4 virt_top4(const float *ch, int n, int t, const uint32_t *const *psp, uint32_t gmask)
{
    constexpr int CNT = 1 << (NV - 1);
    const int s = n - NV;
    const int half = 1 << (n - 1);
    float4 v[CNT];
#pragma unroll
    for (int j = 0; j < CNT; ++j) {
        const int x = t + (j << s);
        const float4 A = *reinterpret_cast<const float4 *>(ch + x);
        const float4 B = *reinterpret_cast<const float4 *>(ch + x + half);
        v[j] = ((gmask >> (NV - 1)) & 1u) ? g4(A, B, psp[NV - 1][x >> 5] >> (x & 31)) : f4(A, B, FEX);
    }
#pragma unroll
    for (int d = NV - 2; d >= 0; --d) {
        const int c = 1 << d;
#pragma unroll
        for (int j = 0; j < c; ++j) {
            const int x = t + (j << s);
            v[j] = ((gmask >> d) & 1u) ? g4(v[j], v[j + c], psp[d][x >> 5] >> (x & 31)) : f4(v[j], v[j + c], FEX);
        }
    }
    return v[0];
}

// One stored level s (width w = 2^s) from a stored source level (src points at
// its first element), f or g with partial sums pw.
template <bool FEX, bool G>
__device__ __forceinline__ void level_from(float *__restrict__ dst, const float *__restrict__ src, int w,
                                           const uint32_t *__restrict__ pw)
{
    if (w >= 4) {
#pragma unroll 2
        for (int t = 0; t < w; t += 4) {
            const float4 A = *reinterpret_cast<const float4 *>(src + t);
            const float4 B = *reinterpret_cast<const float4 *>(src + w + t);
            float4 o;
            if (G) {
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
        const uint32_t bits = G ? pw[0] : 0u;
        for (int t = 0; t < w; ++t)
            dst[t] = G ? scl_g(src[t], src[w + t], (bits >> t) & 1u) : scl_f<FEX>(src[t], src[w + t]);
    }
}

} // namespace pc
