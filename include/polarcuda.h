/*
 * polarcuda.h -- C-ABI of the B200 hybrid BP -> SCL polar decoder.
 *
 * The reference (`polarsim`, /root/reference/pkg/src/polarsim) has no FFI;
 * its seams are Python calls.  Each entry point below replaces one of them
 * (SURVEY.md section 8b):
 *
 *   pc_bp_decode   <- bp.bp_decode            bp.py:194-217 (per frame, here batched)
 *                     + stopping_check        bp.py:176-191 (fused CRC verdict)
 *   pc_bp_iterate  <- bp.iterate_once         bp.py:138-161 (teacher-forced parity hook)
 *   pc_compact     <- hybrid routing          hybrid.py:218-226 (`if draft.converged ... else buffer.put`)
 *   pc_scl_decode  <- _kernels.scl_decode_kernel _kernels.py:144-333
 *                     + winner rule           scl.py:177-191 (CRC-aided, (metric, slot) order)
 *   pc_encode      <- insert_message + polar_transform  polar.py:79-103, 289-306
 *   pc_gen_frames  <- sim._make_frame         sim.py:117-121 (Philox instead of PCG64:
 *                     statistically equivalent only)
 *   pc_count_errors<- sim error counting      sim.py:220-224
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless stated otherwise;
 *     configuration structs are passed by host pointer and read at call time;
 *   - calls are asynchronous and ordered on `stream` (a cudaStream_t, or NULL
 *     for the legacy default stream);
 *   - return 0 on success, a negative PC_ERR_* code otherwise; pc_strerror()
 *     names it.  No exception crosses the ABI;
 *   - bit vectors are packed little-endian in 32-bit words: bit b of a vector
 *     lives in word b/32 at bit position b%32;
 *   - the library keeps no global mutable state; scratch comes from the
 *     caller's workspace (pc_workspace_bytes()).
 */
#ifndef POLARCUDA_H
#define POLARCUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PC_OK 0
#define PC_ERR_INVALID (-1)     /* bad argument (sizes, modes, null pointer) */
#define PC_ERR_UNSUPPORTED (-2) /* configuration outside the compiled kernel set */
#define PC_ERR_CUDA (-3)        /* a CUDA runtime call failed */
#define PC_ERR_NO_DEVICE (-4)   /* no sm_100 device visible */

#define PC_MAX_LOGN 12 /* N <= 4096 (N = 4096 BP: register/shuffle kernel, 512 threads per frame) */
#define PC_MAX_LIST 32

/* A polar code, described by device-resident tables built on the host from
 * CodeConfig (paper_1609_09358_b200/codes.py).  Mirrors polar.py:216-286. */
typedef struct pc_code {
    int32_t N, n, k, m;          /* block length, log2 N, non-frozen count, payload bits */
    int32_t crc_width;           /* 0 (no CRC), 8, 16 or 24 */
    uint32_t crc_offset;         /* CRC register after k zero bits (0 for init = 0) */
    uint32_t enc_crc_offset;     /* CRC register after m zero bits */
    int32_t first_info;          /* info_pos[0], DERIVED by pc_code_seal (SCL decodes the
                                    all-frozen prefix before it element-parallel) */
    const uint32_t *frozen_bits; /* [ceil(N/32)]  1 = frozen                      */
    const uint32_t *crc_cols;    /* [N] register contribution of a 1 at position i */
    const int32_t *info_pos;     /* [k] ascending non-frozen positions             */
    const uint32_t *enc_cols;    /* [m] register contribution of payload bit j     */
    const uint32_t *da_bits;     /* [ceil(N/32)] decision-aided positions or NULL  */
    uint64_t seal;               /* written by pc_code_seal; every decode call checks it */
} pc_code_t;

/* Validate a code's device tables and seal the struct (call once after filling
 * it, before any decode; synchronous on `stream`).  Reads frozen_bits, info_pos
 * and da_bits back and checks: N - k frozen positions; info_pos = the
 * non-frozen positions in ascending order; decision-aided positions are not
 * frozen.  Then DERIVES first_info = info_pos[0] (the caller's value is
 * ignored) and writes `seal`, a hash of every field.  pc_bp_decode,
 * pc_bp_iterate, pc_scl_decode, pc_encode and pc_gen_frames return
 * PC_ERR_INVALID for a struct that was never sealed or was changed after
 * sealing (e.g. a hand-set first_info), instead of decoding with it.
 * Mirrors the validation of CodeConfig.__init__ (polar.py:235-263). */
int pc_code_seal(pc_code_t *code, void *stream);

/* BpConfig, bp.py:40-57.  g_mode 0 = exact (likelihood-ratio arithmetic:
 * messages e^v, g = (1 + xy)/(x + y), one reciprocal per g), 1 = min, 2 = exact
 * evaluated per g (4 MUFU, natural log domain; N = 1024/2048, parity studies),
 * 3 = exact in the round-1 exponential/log2 form (2.875 MUFU per g; register/
 * shuffle kernel only, N = 128..4096; an A/B knob); stop_mode 0 = crc,
 * 1 = reencode, 2 = none.  threads_per_frame 0 = library default.
 * kernel: 0 = auto (register/shuffle kernel when eligible), 1 = shared-memory
 * kernel, 2 = register/shuffle kernel (N = 128..4096, every stop rule, the
 * re-encode stop with threads_per_frame >= 64; soft_x only at N = 4096, which
 * runs only on this kernel); a performance knob: both kernels restate the same
 * fp64 recursion in fp32 and may part only on certified near-ties. */
typedef struct pc_bp_cfg {
    int32_t i_max, g_mode, stop_mode, threads_per_frame;
    float llr_max;
    int32_t kernel;
    /* Optional 4 bytes of device scratch, private to this call's stream: the
     * frame counter of the persistent register/shuffle kernel (one CTA per
     * resident slot, frames taken from the counter; 14% faster at N = 128,
     * where frames of 1..i_max iterations otherwise leave CTA slots empty).
     * NULL = one CTA per frame.  Does not change results. */
    int32_t *work;
} pc_bp_cfg_t;

/* SclConfig, scl.py:39-66.  L in 1..32 (N >= 64 for L not a power of two: the
 * v3 kernel keeps L paths on the next power of two of lanes).  virtual_levels: how many of
 * the top tree levels are recomputed from the channel instead of stored
 * (-1 = library default); a performance knob that does not change results.
 * warps_per_cta: 1..4 (0 = 1).  kernel: 0 = auto (L = 1 and N >= 64: the
 * one-warp-per-frame SC kernel; else the v3 register-block kernel for N >= 64,
 * else v2), 1 = v2 (per-leaf shared-memory kernel), 2 = v3, 3 = the SC kernel
 * (L = 1 only); performance knobs that do not change results. */
typedef struct pc_scl_cfg {
    int32_t L, metric_exact, f_exact, selector_bitonic, virtual_levels, warps_per_cta;
    int32_t kernel;
} pc_scl_cfg_t;

int pc_version(void);
const char *pc_strerror(int code);
/* Bytes of device scratch the decode calls need (counters, queue heads). */
int64_t pc_workspace_bytes(void);
/* Number of visible devices with compute capability 10.x (0 on a CPU host). */
int pc_device_count(void);

/* Batched BP decode (bp_decode, bp.py:194-217) with the stop rule evaluated
 * after every iteration (bp.py:203-208).
 *   llr        [B][N] fp32 channel LLRs
 *   u_bits     [B][ceil(N/32)] hard decisions u_hat        (nullable)
 *   payload    [B][ceil(m/32)] u_hat[info_pos[0..m-1]]     (nullable)
 *   soft_u     [B][N] L0 + R0 at exit                      (nullable)
 *   soft_x     [B][N] Ln + Rn at exit                      (nullable)
 *   iters      [B] iterations_used (i_max when not converged)
 *   converged  [B] 1 when the stop rule fired
 *   t_done     [B] %globaltimer (ns) when the frame's decision was final (nullable) */
int pc_bp_decode(const float *llr, int32_t B, const pc_code_t *code, const pc_bp_cfg_t *cfg, uint32_t *u_bits,
                 uint32_t *payload, float *soft_u, float *soft_x, int32_t *iters, uint8_t *converged,
                 uint64_t *t_done, void *stream);

/* One full BP iteration (R sweep, L sweep) in place on explicit state
 * l_msgs, r_msgs [B][n+1][N] (bp.py:138-161): the teacher-forced parity hook. */
int pc_bp_iterate(float *l_msgs, float *r_msgs, int32_t B, const pc_code_t *code, const pc_bp_cfg_t *cfg,
                  void *stream);

/* Failed-frame stream compaction: queue <- { b : converged[b] == 0 },
 * *count <- |queue| (device int32).  Queue order is unspecified; results
 * written per frame index do not depend on it. */
int pc_compact(const uint8_t *converged, int32_t B, int32_t *queue, int32_t *count, void *workspace, void *stream);

/* Bytes of device workspace pc_scl_decode needs for this code and
 * configuration (counters + the K3 decision traceback); -1 on bad arguments. */
int64_t pc_scl_workspace_bytes(const pc_code_t *code, const pc_scl_cfg_t *cfg);

/* Batched SCL decode with the CRC-aided winner (scl.py:151-197).
 * workspace: at least pc_scl_workspace_bytes(code, cfg) bytes of device memory.
 * Frames decoded: queue[0..*count-1] (queue, count device) or 0..B-1 when
 * queue is NULL.  Outputs are indexed by FRAME, so the hybrid writes them
 * into the same per-frame arrays as pc_bp_decode.
 *   u_bits [B][ceil(N/32)], payload [B][ceil(m/32)] (nullable each),
 *   metric [B] winner metric (nullable), crc_ok [B] (nullable),
 *   sel_by_crc [B] (nullable), t_done [B] (nullable). */
int pc_scl_decode(const float *llr, int32_t B, const int32_t *queue, const int32_t *count, const pc_code_t *code,
                  const pc_scl_cfg_t *cfg, uint32_t *u_bits, uint32_t *payload, float *metric, uint8_t *crc_ok,
                  uint8_t *sel_by_crc, uint64_t *t_done, void *workspace, void *stream);

/* Encoder (insert_message + polar_transform): msg_bits [B][ceil(m/32)] ->
 * x_bits [B][ceil(N/32)].  Bit-exact hook for the encoder/CRC contract. */
int pc_encode(const uint32_t *msg_bits, int32_t B, const pc_code_t *code, uint32_t *x_bits, void *stream);

/* Device frame generator: Philox-4x32-10 keyed by (seed, point, frame0 + b)
 * draws the payload and the AWGN; writes msg_bits [B][ceil(m/32)] and
 * llr [B][N] = 2 (1 - 2x + sigma w) / sigma^2 (sigma = 0: +/-20 saturated). */
int pc_gen_frames(uint64_t seed, int32_t point, int64_t frame0, int32_t B, float sigma, const pc_code_t *code,
                  uint32_t *msg_bits, float *llr, void *stream);

/* Error counting on payload bits (sim.py:220-224): counters[0] += bit errors,
 * counters[1] += frame errors (int64, device). */
int pc_count_errors(const uint32_t *payload, const uint32_t *msg_bits, int32_t B, int32_t m, int64_t *counters,
                    void *stream);

/* Latency helper: writes %globaltimer (ns) to *t (device) on `stream`. */
int pc_stamp(uint64_t *t, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* POLARCUDA_H */
