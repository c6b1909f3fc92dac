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

} // namespace pc
