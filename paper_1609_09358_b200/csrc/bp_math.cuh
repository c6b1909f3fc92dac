// bp_math.cuh -- the BP node update shared by K1 (v1 and v2) and the parity hook.
#pragma once
#include "common.cuh"

namespace pc {

__device__ __forceinline__ float sp_neg(float x) // log1p(exp(-x)), x >= 0
{
    return PC_LN2 * lg2_approx(1.0f + ex2_approx(-x * PC_LOG2E));
}

template <int GMODE>
__device__ __forceinline__ float bp_g(float a, float b, float lim)
{
    const float aa = fabsf(a), ab = fabsf(b);
    const float m = fminf(aa, ab);
    float mag;
    if (GMODE == 0) {
        mag = m + sp_neg(aa + ab) - sp_neg(fabsf(aa - ab));
        mag = fminf(fmaxf(mag, 0.0f), m);
    } else {
        mag = (a == 0.0f || b == 0.0f) ? 0.0f : m;
    }
    (void)lim; // |g| <= min(|a|,|b|) and the first argument is always a clipped message
    const uint32_t sgn = (__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u;
    return __uint_as_float(__float_as_uint(mag) ^ sgn);
}

// Both node updates of one processing element share an operand x (bp.py:145-158):
//   R sweep  x = a,  y1 = l2 + r2, y2 = l1, add = r2:  o1 = g(a, l2 + r2),  o2 = clip(g(a, l1) + r2)
//   L sweep  x = l1, y1 = l2 + r2, y2 = a,  add = l2:  o1 = g(l1, l2 + r2), o2 = clip(g(a, l1) + l2)
// Exact g in the exponential domain, p = e^-|v| in (0, 1]:
//   |g(x, y)| = ln(1 + px py) - ln(px + py)            (= logaddexp(0, x+y) - logaddexp(x, y), bp.py:95)
// so a PE costs 3 EX2 + 4 LG2 on the MUFU pipe (px shared) instead of 8.  The
// magnitude is floored at lb (m = min(|x|, |y|), M = max).  The difference of two
// fp32 logs has an absolute error near 1e-7 and would flush tiny exact values
// (|g| ~ m tanh(M/2) for m -> 0) to 0; lb = min(m, 2^-10) (2 - X) / 2, X = 1 + px py,
// keeps their sign and first-order magnitude (an
// absolute deviation below 2^-20 from the exact value; tools/bp_formula_study.py).
// Message domains.  The node-update mode GMODE equals pc_bp_cfg_t.g_mode:
//   0  exact g in the LIKELIHOOD-RATIO domain (default): a message is
//      Lambda = e^v.  A sum of LLRs is a product, the exact node update is
//          g = (1 + Lx Ly) / (Lx + Ly)                    (bp.py:86-100)
//      (one MUFU.RCP per g, no exp/log), the clip |v| <= llr_max is a clamp
//      to [e^-llr_max, e^llr_max] and a hard decision is Lambda < 1.  The
//      clip keeps every message in [e^-20, e^20] (sums up to e^40), far inside
//      fp32; the price is absolute (not relative) resolution near v = 0
//      (about 6e-8), the same order as the log-domain form's cancellation
//      error (tools/lr_domain_study.py: same parity class as g_mode 3);
//   1  min-sum, natural LLR units (bit-identical to an fp32 restatement);
//   2  exact g evaluated per g in natural LLR units (4 MUFU; parity studies);
//   3  exact g in the exponential domain of the round-1 kernel, messages in
//      log2 units (LLR * log2 e), 2.875 MUFU per g (A/B knob).
// Every kernel uses the helpers below for init, sums, decisions, clip and
// conversions, so a mode's arithmetic is the same in K1 v1, K1 v2 and the
// teacher-forced hook.
template <int GMODE>
__host__ __device__ constexpr float bp_unit_in() { return (GMODE == 0 || GMODE == 3) ? PC_LOG2E : 1.0f; }
template <int GMODE>
__host__ __device__ constexpr float bp_unit_out() { return (GMODE == 0 || GMODE == 3) ? PC_LN2 : 1.0f; }

__device__ __forceinline__ float rcp_approx(float x)
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct BpLim { // clip bounds in message units
    float hi, lo;
};
template <int GMODE>
__device__ __forceinline__ BpLim bp_lim(float llr_max)
{
    const float u = llr_max * bp_unit_in<GMODE>();
    return GMODE == 0 ? BpLim{ex2_approx(u), ex2_approx(-u)} : BpLim{u, -u};
}
template <int GMODE>
__device__ __forceinline__ float bp_clip(float v, BpLim l) { return fminf(fmaxf(v, l.lo), l.hi); }
template <int GMODE>
__device__ __forceinline__ float bp_zero() { return GMODE == 0 ? 1.0f : 0.0f; } // the LLR 0
template <int GMODE>
__device__ __forceinline__ float bp_comb(float a, float b) { return GMODE == 0 ? a * b : a + b; } // LLR a + b
template <int GMODE>
__device__ __forceinline__ bool bp_neg(float v) { return GMODE == 0 ? v < 1.0f : v < 0.0f; } // LLR < 0: bit 1
// channel LLR (natural units) -> clipped message; message -> natural LLR
template <int GMODE>
__device__ __forceinline__ float bp_load(float llr, float llr_max)
{
    const float u = llr_max * bp_unit_in<GMODE>();
    const float v = fminf(fmaxf(llr * bp_unit_in<GMODE>(), -u), u);
    return GMODE == 0 ? ex2_approx(v) : v;
}
template <int GMODE>
__device__ __forceinline__ float bp_store(float m) { return GMODE == 0 ? lg2_approx(m) * PC_LN2 : m * bp_unit_out<GMODE>(); }
// the frozen prior R[0] = llr_max (bp.py:133)
template <int GMODE>
__device__ __forceinline__ float bp_prior(BpLim l) { return l.hi; }

// The exponential of the PE's sum operand (l2 + r2) runs on the FMA pipe
// (ex2_fma): the kernel is XU-bound with issue slots to spare.
#ifndef BP_EX2_Y1
#define BP_EX2_Y1 ex2_fma
#endif
#ifndef BP_EX2_Y1L
#define BP_EX2_Y1L ex2_approx
#endif

// Core of a PE update with the three exponentials p = 2^-|v| given (GMODE 3).
__device__ __forceinline__ void bp_pe2_core(float x, float y1, float y2, float px, float p1, float p2, float add,
                                            BpLim lim, float &o1, float &o2)
{
    const float ax = fabsf(x), a1 = fabsf(y1), a2 = fabsf(y2);
    const float X1 = fmaf(px, p1, 1.0f), X2 = fmaf(px, p2, 1.0f);
    float m1 = lg2_approx(X1) - lg2_approx(px + p1); // log2 units: |g'| = lg2(1 + px py) - lg2(px + py)
    float m2 = lg2_approx(X2) - lg2_approx(px + p2);
    // (no upper clamp at min(|x|, |y|): the computed value exceeds it by rounding
    // noise only, and every message is clipped or feeds a clipped one)
    const float lb1 = fminf(fminf(ax, a1), 0.0009765625f) * fmaf(-0.5f, X1, 1.0f);
    const float lb2 = fminf(fminf(ax, a2), 0.0009765625f) * fmaf(-0.5f, X2, 1.0f);
    m1 = fmaxf(m1, lb1);
    m2 = fmaxf(m2, lb2);
    o1 = __uint_as_float(__float_as_uint(m1) ^ ((__float_as_uint(x) ^ __float_as_uint(y1)) & 0x80000000u));
    const float g2 = __uint_as_float(__float_as_uint(m2) ^ ((__float_as_uint(x) ^ __float_as_uint(y2)) & 0x80000000u));
    o2 = bp_clip<3>(g2 + add, lim);
}

// RS: an R-sweep PE (the sum operand's exponential on the FMA pipe) or an
// L-sweep PE (on the MUFU) -- the same choice as bp_pe2_keep / bp_pe2_p2, so a
// PE's arithmetic never depends on which boundaries keep their exponentials.
// LFMA: the L sweep also uses the FMA pipe (kernels without kept exponentials,
// N = 4096, where the MUFU has one more op per L-sweep PE to shed).
template <int GMODE, bool RS, bool LFMA = false>
__device__ __forceinline__ void bp_pe2(float x, float y1, float y2, float add, BpLim lim, float &o1, float &o2)
{
    if (GMODE == 0) { // likelihood ratios: g = (1 + x y) / (x + y)
        // (one reciprocal of (x + y1)(x + y2) for both quotients measured no faster:
        // -0.6% at N=1024, tools/k1_variant_probe.sh; the kernel is issue-bound)
        o1 = fmaf(x, y1, 1.0f) * rcp_approx(x + y1);
        o2 = bp_clip<0>(fmaf(x, y2, 1.0f) * rcp_approx(x + y2) * add, lim);
        return;
    }
    if (GMODE == 2) {
        o1 = bp_g<0>(x, y1, lim.hi);
        o2 = bp_clip<2>(bp_g<0>(x, y2, lim.hi) + add, lim);
        return;
    }
    if (GMODE == 3) { // log2 units: p = 2^-|v'|
        bp_pe2_core(x, y1, y2, ex2_approx(-fabsf(x)),
                    (RS || LFMA) ? BP_EX2_Y1(-fabsf(y1)) : BP_EX2_Y1L(-fabsf(y1)), ex2_approx(-fabsf(y2)), add, lim,
                    o1, o2);
        return;
    }
    const float ax = fabsf(x), a1 = fabsf(y1), a2 = fabsf(y2);
    const float m1 = (x == 0.0f || y1 == 0.0f) ? 0.0f : fminf(ax, a1);
    const float m2 = (x == 0.0f || y2 == 0.0f) ? 0.0f : fminf(ax, a2);
    o1 = __uint_as_float(__float_as_uint(m1) ^ ((__float_as_uint(x) ^ __float_as_uint(y1)) & 0x80000000u));
    const float g2 = __uint_as_float(__float_as_uint(m2) ^ ((__float_as_uint(x) ^ __float_as_uint(y2)) & 0x80000000u));
    o2 = bp_clip<1>(g2 + add, lim);
}

// GMODE 3 R-sweep PE that also returns px = 2^-|a| (x = a) for reuse by the
// L sweep at the same boundary, where a is the second operand (bp_pe2_p2).
__device__ __forceinline__ void bp_pe2_keep(float x, float y1, float y2, float add, BpLim lim, float &o1, float &o2,
                                            float &px)
{
    px = ex2_approx(-fabsf(x));
    bp_pe2_core(x, y1, y2, px, BP_EX2_Y1(-fabsf(y1)), ex2_approx(-fabsf(y2)), add, lim, o1, o2);
}

// GMODE 3 L-sweep PE with p2 = 2^-|y2| supplied (y2 = a, kept from the R sweep).
__device__ __forceinline__ void bp_pe2_p2(float x, float y1, float y2, float p2, float add, BpLim lim, float &o1,
                                          float &o2)
{
    bp_pe2_core(x, y1, y2, ex2_approx(-fabsf(x)), BP_EX2_Y1L(-fabsf(y1)), p2, add, lim, o1, o2);
}

} // namespace pc
