// aux.cu -- K2 compaction, K4 encoder / frame generator, error counting.
#include "common.cuh"

namespace pc {

// ------------------------------------------------------------ K2 compact --
// hybrid.py:218-226 routes every BP failure to the list decoder; here a
// warp-aggregated atomic appends failed frame indices to a dense queue.
__global__ void k_compact(const uint8_t *__restrict__ conv, int B, int32_t *queue, int32_t *count)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    const bool fail = b < B && conv[b] == 0;
    const uint32_t m = __ballot_sync(0xffffffffu, fail);
    if (m == 0)
        return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader)
        base = atomicAdd(count, __popc(m));
    // every lane of the warp reaches this point (the m == 0 exit above is warp-uniform)
    base = __shfl_sync(0xffffffffu, base, leader);
    if (fail)
        queue[base + __popc(m & ((1u << lane) - 1u))] = b;
}

// --------------------------------------------------- Philox-4x32-10 (K4) --
struct u4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ u4 philox(u4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = u4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// Encode one frame held as bits in shared memory: payload -> u (payload,
// CRC at info positions) -> x = u F^{(x)n}.  polar.py:79-103, 289-306.
// `msg` holds ceil(m/32) words, `u` receives ceil(N/32) words.
__device__ void encode_block(const Code &c, const uint32_t *msg, uint32_t *u, uint32_t *scratch)
{
    const int NW = (c.N + 31) >> 5;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int w = tid; w < NW; w += nt)
        u[w] = 0u;
    // CRC register of the payload through the affine encoder table
    uint32_t syn = 0;
    for (int j = tid; j < c.m; j += nt)
        if (bit_of(msg, j))
            syn ^= __ldg(c.enc_cols + j);
    syn = __reduce_xor_sync(0xffffffffu, syn);
    if ((tid & 31) == 0)
        scratch[tid >> 5] = syn;
    __syncthreads();
    uint32_t reg = c.enc_crc_offset;
    for (int w = 0; w < (nt + 31) / 32; ++w)
        reg ^= scratch[w];
    for (int j = tid; j < c.k; j += nt) {
        const uint32_t bit = j < c.m ? bit_of(msg, j) : (reg >> (c.crc_width - 1 - (j - c.m))) & 1u;
        if (bit) {
            const int pos = __ldg(c.info_pos + j);
            atomicOr(u + (pos >> 5), 1u << (pos & 31));
        }
    }
    __syncthreads();
    // butterfly stages inside a word (h = 1..16) ...
    const uint32_t masks[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
    for (int w = tid; w < NW; w += nt) {
        uint32_t v = u[w];
        for (int s = 0; s < 5 && (1 << s) < c.N; ++s)
            v ^= (v >> (1 << s)) & masks[s];
        u[w] = v;
    }
    __syncthreads();
    // ... and across words (h = 32, 64, ...)
    for (int H = 1; H < NW; H <<= 1) {
        for (int w = tid; w < NW; w += nt)
            if ((w & H) == 0)
                u[w] ^= u[w + H];
        __syncthreads();
    }
}

struct GenArgs {
    Code c;
    uint64_t seed;
    int32_t point;
    int64_t frame0;
    int32_t B;
    float sigma;
    uint32_t *msg_bits;
    float *llr;
};

__global__ void __launch_bounds__(128) k_gen(const GenArgs a)
{
    __shared__ uint32_t msg[128];   // up to 4096 payload bits
    __shared__ uint32_t u[128];     // up to N = 4096
    __shared__ uint32_t scratch[8];
    const int b = blockIdx.x;
    const int64_t frame = a.frame0 + b;
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32) ^ (0x85EBCA6Bu * (uint32_t)a.point);
    const int MW = (a.c.m + 31) >> 5, NW = (a.c.N + 31) >> 5;
    // payload bits: counter stream 1
    for (int g = threadIdx.x; g * 4 < MW; g += blockDim.x) {
        const u4 r = philox(u4{(uint32_t)g, (uint32_t)frame, (uint32_t)(frame >> 32), 1u}, k0, k1);
        const uint32_t vals[4] = {r.x, r.y, r.z, r.w};
        for (int e = 0; e < 4 && 4 * g + e < MW; ++e) {
            const int w = 4 * g + e;
            uint32_t v = vals[e];
            if (32 * w + 32 > a.c.m)
                v &= (1u << (a.c.m & 31)) - 1u;
            msg[w] = v;
        }
    }
    __syncthreads();
    if (a.msg_bits != nullptr)
        for (int w = threadIdx.x; w < MW; w += blockDim.x)
            a.msg_bits[(size_t)b * MW + w] = msg[w];
    encode_block(a.c, msg, u, scratch);
    // noise: counter stream 2, Box-Muller on pairs
    const float s = a.sigma;
    const float scale = s > 0.0f ? 2.0f / (s * s) : 0.0f;
    for (int g = threadIdx.x; 4 * g < a.c.N; g += blockDim.x) {
        const u4 r = philox(u4{(uint32_t)g, (uint32_t)frame, (uint32_t)(frame >> 32), 2u}, k0, k1);
        const float u1 = ((r.x >> 8) + 1) * (1.0f / 16777216.0f), u2 = (r.y >> 8) * (1.0f / 16777216.0f);
        const float u3 = ((r.z >> 8) + 1) * (1.0f / 16777216.0f), u4f = (r.w >> 8) * (1.0f / 16777216.0f);
        const float rad1 = sqrtf(-2.0f * logf(u1)), rad2 = sqrtf(-2.0f * logf(u3));
        float sn1, cs1, sn2, cs2;
        sincospif(2.0f * u2, &sn1, &cs1);
        sincospif(2.0f * u4f, &sn2, &cs2);
        const float z[4] = {rad1 * cs1, rad1 * sn1, rad2 * cs2, rad2 * sn2};
        for (int e = 0; e < 4 && 4 * g + e < a.c.N; ++e) {
            const int i = 4 * g + e;
            const float sym = bit_of(u, i) ? -1.0f : 1.0f;
            a.llr[(size_t)b * a.c.N + i] = s > 0.0f ? scale * (sym + s * z[e]) : 20.0f * sym;
        }
    }
}

__global__ void __launch_bounds__(128) k_encode(Code c, const uint32_t *msg_bits, int B, uint32_t *x_bits)
{
    __shared__ uint32_t msg[128];
    __shared__ uint32_t u[128];
    __shared__ uint32_t scratch[8];
    const int b = blockIdx.x;
    const int MW = (c.m + 31) >> 5, NW = (c.N + 31) >> 5;
    for (int w = threadIdx.x; w < MW; w += blockDim.x)
        msg[w] = msg_bits[(size_t)b * MW + w];
    __syncthreads();
    encode_block(c, msg, u, scratch);
    for (int w = threadIdx.x; w < NW; w += blockDim.x) {
        uint32_t v = u[w];
        if (32 * w + 32 > c.N)
            v &= (1u << (c.N & 31)) - 1u;
        x_bits[(size_t)b * NW + w] = v;
    }
}

// ---------------------------------------------------------- error counts --
__global__ void k_count_errors(const uint32_t *pay, const uint32_t *msg, int B, int m, unsigned long long *cnt)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long be = 0, fe = 0;
    if (b < B) {
        const int MW = (m + 31) >> 5;
        int e = 0;
        for (int w = 0; w < MW; ++w) {
            uint32_t d = pay[(size_t)b * MW + w] ^ msg[(size_t)b * MW + w];
            if (32 * w + 32 > m)
                d &= (1u << (m & 31)) - 1u;
            e += __popc(d);
        }
        be = e;
        fe = e > 0;
    }
    for (int off = 16; off; off >>= 1) {
        be += __shfl_xor_sync(0xffffffffu, be, off);
        fe += __shfl_xor_sync(0xffffffffu, fe, off);
    }
    if ((threadIdx.x & 31) == 0 && (be | fe)) {
        atomicAdd(cnt, be);
        atomicAdd(cnt + 1, fe);
    }
}

__global__ void k_stamp(uint64_t *t) { *t = globaltimer(); }

// ------------------------------------------------------------- launchers --
int launch_compact(const uint8_t *conv, int B, int32_t *queue, int32_t *count, cudaStream_t s)
{
    if (cudaMemsetAsync(count, 0, sizeof(int32_t), s) != cudaSuccess)
        return PC_ERR_CUDA;
    if (B == 0)
        return PC_OK;
    k_compact<<<(B + 255) / 256, 256, 0, s>>>(conv, B, queue, count);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

int launch_gen(const Code &c, uint64_t seed, int point, int64_t frame0, int B, float sigma, uint32_t *msg, float *llr,
               cudaStream_t s)
{
    if (B == 0)
        return PC_OK;
    GenArgs a{c, seed, point, frame0, B, sigma, msg, llr};
    k_gen<<<B, 128, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

int launch_encode(const Code &c, const uint32_t *msg, int B, uint32_t *x, cudaStream_t s)
{
    if (B == 0)
        return PC_OK;
    k_encode<<<B, 128, 0, s>>>(c, msg, B, x);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

int launch_count_errors(const uint32_t *pay, const uint32_t *msg, int B, int m, int64_t *cnt, cudaStream_t s)
{
    if (B == 0)
        return PC_OK;
    k_count_errors<<<(B + 255) / 256, 256, 0, s>>>(pay, msg, B, m, reinterpret_cast<unsigned long long *>(cnt));
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

int launch_stamp(uint64_t *t, cudaStream_t s)
{
    k_stamp<<<1, 1, 0, s>>>(t);
    return cudaGetLastError() == cudaSuccess ? PC_OK : PC_ERR_CUDA;
}

} // namespace pc
