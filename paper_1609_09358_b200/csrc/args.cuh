// args.cuh -- kernel argument blocks shared by the launchers and the C-ABI.
#pragma once
#include "common.cuh"

namespace pc {

struct BpArgs {
    const float *llr;
    int32_t B;
    Code code;
    int32_t i_max, stop_mode;
    float llr_max;
    uint32_t *u_bits, *payload;
    float *soft_u, *soft_x;
    int32_t *iters;
    uint8_t *conv;
    uint64_t *t_done;
    int32_t *work; // frame counter of the persistent K1 variant (nullptr: one CTA per frame)
};

struct SclArgs {
    const float *llr;
    int32_t B;
    const int32_t *queue, *count;
    Code code;
    int32_t metric_exact, f_exact;
    int32_t list_cap; // the list size L (K3 v3 runs it on the next power of two of lanes)
    int32_t nv;       // virtual top levels
    uint32_t *u_bits, *payload;
    float *metric;
    uint8_t *crc_ok, *sel;
    uint64_t *t_done;
    int32_t *work; // persistent-warp work counter
    // derived layout (per warp, in 32-bit words)
    int32_t tp;      // top stored LLR level
    int32_t ss;      // LLR slot stride (floats)
    int32_t psw;     // partial-sum slot stride (words)
    int32_t uhs;     // decision slot stride (words)
    int32_t warp_words;  // per-warp shared words (slots, partial sums, decisions, candidates, channel)
    int32_t table_words; // CTA-shared frozen / decision-aided masks
    // v3 (scl3.cu) per-warp section offsets, in 32-bit words from the warp base
    int32_t o_ps, o_tb, o_tba, o_cand, o_wrow, o_ch;
    int32_t prefix; // v3: frozen-prefix fast path enabled (L = 32 and 2N floats of scratch fit)
    uint32_t *tbg;  // v3: decision traceback in the caller's workspace (after the 256-byte counter block)
};

int launch_bp_decode(const BpArgs &a, int g_mode, int tpf, int kernel, cudaStream_t s);
bool bp2_eligible(const BpArgs &a, int g_mode, int tpf);
int launch_bp2(const BpArgs &a, int g_mode, int tpf, cudaStream_t s);
bool bp3_eligible(const BpArgs &a, int g_mode, int tpf);
int launch_bp3(const BpArgs &a, int g_mode, cudaStream_t s);
bool bp3h_eligible(const BpArgs &a, int g_mode, int tpf);
int launch_bp3h(const BpArgs &a, int g_mode, cudaStream_t s);
int launch_bp_iterate(float *l, float *r, int B, int n, int g_mode, float lim, cudaStream_t s);
int scl_prepare(SclArgs &a, int nv_req);
int launch_scl(const SclArgs &a, int L, int wpc, cudaStream_t s);
bool scl3_eligible(const SclArgs &a, int L);
int scl3_prepare(SclArgs &a, int L, int nv_req);
int launch_scl3(const SclArgs &a, int L, int wpc, cudaStream_t s);
int64_t scl3_workspace_bytes(const SclArgs &a, int L, int wpc);
bool sc1_eligible(const SclArgs &a);
int launch_sc1(const SclArgs &a, cudaStream_t s);
int launch_compact(const uint8_t *conv, int B, int32_t *queue, int32_t *count, cudaStream_t s);
int launch_gen(const Code &c, uint64_t seed, int point, int64_t frame0, int B, float sigma, uint32_t *msg, float *llr,
               cudaStream_t s);
int launch_encode(const Code &c, const uint32_t *msg, int B, uint32_t *x, cudaStream_t s);
int launch_count_errors(const uint32_t *pay, const uint32_t *msg, int B, int m, int64_t *cnt, cudaStream_t s);
int launch_stamp(uint64_t *t, cudaStream_t s);

} // namespace pc
