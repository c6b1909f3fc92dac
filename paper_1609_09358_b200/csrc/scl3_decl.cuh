// scl3_decl.cuh -- declarations shared by the K3 v3 host code and its per-L units.
#pragma once
#include "args.cuh"

namespace pc {
namespace s3 {
#ifndef PC_SCL3_T
#define PC_SCL3_T 5
#endif
constexpr int T = PC_SCL3_T; // leaf-block level: 2^T leaves per block (3..5; 5 measured best)
constexpr int BL = 1 << T; // leaves per block
// word offset of partial-sum level s (T <= s <= n-1) inside a slot
__host__ __device__ __forceinline__ int pso(int s) { return s < 5 ? s - T : (5 - T) + (1 << (s - 5)) - 1; }
// float offset of LLR level s (T+1 <= s <= tp) inside a slot
__host__ __device__ __forceinline__ int llo(int s) { return (1 << s) - (1 << (T + 1)); }
} // namespace s3

template <int L>
int launch_scl3_for(const SclArgs &a, int wpc, int max_warps, cudaStream_t s);
} // namespace pc
