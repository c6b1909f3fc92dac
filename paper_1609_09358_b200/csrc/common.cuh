// common.cuh -- device helpers shared by the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "polarcuda.h"

#define PC_LOG2E 1.4426950408889634f
#define PC_LN2 0.6931471805599453f

namespace pc {

// MUFU (XU pipe) approximations; flush-to-zero keeps them single-instruction.
__device__ __forceinline__ float ex2_approx(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float lg2_approx(float x)
{
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x for x in [-126, 0] on the FMA/ALU pipes (no MUFU): x = j + f with j the
// nearest integer (magic-number rounding), f in [-0.5, 0.5]; degree-5
// polynomial for 2^f (relative error < 2.2e-7 in fp32, the same order as
// ex2.approx), then j added to the exponent field.
__device__ __forceinline__ float ex2_fma(float x)
{
    const float t = __fadd_rn(x, 12582912.0f); // 1.5 * 2^23
    const float f = __fsub_rn(x, __fsub_rn(t, 12582912.0f));
    float p = fmaf(0.0013266970636323094f, f, 0.009675459936261177f);
    p = fmaf(p, f, 0.05550742521882057f);
    p = fmaf(p, f, 0.24022121727466583f);
    p = fmaf(p, f, 0.6931469440460205f);
    p = fmaf(p, f, 1.0000001192092896f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// 1-D TMA bulk copy (cp.async.bulk, SASS UBLKCP) global -> shared memory,
// completing on an mbarrier: one elected thread arms the barrier with the byte
// count and issues the copy; every thread then waits on the barrier's phase.
// dst / src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(mbar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *mbar)
{
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t phase)
{
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(mbar);
    asm volatile("{\n\t.reg .pred p;\n"
                 "WAIT%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT%=;\n}" ::"r"(b),
                 "r"(phase)
                 : "memory");
}

__device__ __forceinline__ uint64_t globaltimer()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ float clampf(float v, float lim) { return fminf(fmaxf(v, -lim), lim); }

__device__ __forceinline__ uint32_t bit_of(const uint32_t *words, int i) { return (words[i >> 5] >> (i & 31)) & 1u; }

// Device copy of pc_code_t (same layout; kernels take it by value).
struct Code {
    int32_t N, n, k, m, crc_width;
    uint32_t crc_offset, enc_crc_offset;
    int32_t first_info;
    const uint32_t *frozen_bits, *crc_cols;
    const int32_t *info_pos;
    const uint32_t *enc_cols, *da_bits;
};

inline Code to_device_code(const pc_code_t &c)
{
    Code d;
    d.N = c.N;
    d.n = c.n;
    d.k = c.k;
    d.m = c.m;
    d.crc_width = c.crc_width;
    d.crc_offset = c.crc_offset;
    d.enc_crc_offset = c.enc_crc_offset;
    d.first_info = c.first_info;
    d.frozen_bits = c.frozen_bits;
    d.crc_cols = c.crc_cols;
    d.info_pos = c.info_pos;
    d.enc_cols = c.enc_cols;
    d.da_bits = c.da_bits;
    return d;
}

} // namespace pc
