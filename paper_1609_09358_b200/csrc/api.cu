// api.cu -- the C-ABI (include/polarcuda.h): validation, then the launchers.
#include "args.cuh"

#include <vector>

using namespace pc;

// Hash of every field a kernel reads (not the seal itself), salted so that a
// zero-filled struct never carries a valid seal.
static uint64_t seal_of(const pc_code_t *c)
{
    uint64_t h = 0xcbf29ce484222325ull ^ 0x706f6c6172637564ull;
    auto mix = [&h](uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (8 * i)) & 0xffu;
            h *= 0x100000001b3ull;
        }
    };
    mix((uint32_t)c->N), mix((uint32_t)c->n), mix((uint32_t)c->k), mix((uint32_t)c->m);
    mix((uint32_t)c->crc_width), mix(c->crc_offset), mix(c->enc_crc_offset), mix((uint32_t)c->first_info);
    mix((uintptr_t)c->frozen_bits), mix((uintptr_t)c->crc_cols), mix((uintptr_t)c->info_pos);
    mix((uintptr_t)c->enc_cols), mix((uintptr_t)c->da_bits);
    return h | 1u;
}

static int check_shape(const pc_code_t *c)
{
    if (c == nullptr || c->N < 2 || c->n < 1 || c->n > PC_MAX_LOGN || (1 << c->n) != c->N)
        return PC_ERR_INVALID;
    if (c->k < 1 || c->k > c->N || c->m < 0 || c->m != c->k - c->crc_width)
        return PC_ERR_INVALID;
    if (c->crc_width != 0 && c->crc_width != 8 && c->crc_width != 16 && c->crc_width != 24)
        return PC_ERR_INVALID;
    if (c->frozen_bits == nullptr || c->info_pos == nullptr)
        return PC_ERR_INVALID;
    if (c->first_info < 0 || c->first_info >= c->N)
        return PC_ERR_INVALID;
    return PC_OK;
}

static int check_code(const pc_code_t *c)
{
    const int rc = check_shape(c);
    if (rc)
        return rc;
    return c->seal == seal_of(c) ? PC_OK : PC_ERR_INVALID; // never sealed, or changed since
}

extern "C" {

int pc_version(void) { return 1; }

int pc_code_seal(pc_code_t *code, void *stream)
{
    if (code == nullptr)
        return PC_ERR_INVALID;
    code->first_info = 0; // derived below; the shape check must not depend on the caller's value
    int rc = check_shape(code);
    if (rc)
        return rc;
    const int N = code->N, k = code->k, NW = (N + 31) / 32;
    std::vector<uint32_t> fz(NW), da;
    std::vector<int32_t> ip(k);
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemcpyAsync(fz.data(), code->frozen_bits, NW * sizeof(uint32_t), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess ||
        cudaMemcpyAsync(ip.data(), code->info_pos, k * sizeof(int32_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return PC_ERR_CUDA;
    if (code->da_bits != nullptr) {
        da.resize(NW);
        if (cudaMemcpyAsync(da.data(), code->da_bits, NW * sizeof(uint32_t), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess)
            return PC_ERR_CUDA;
    }
    if (cudaStreamSynchronize(s) != cudaSuccess)
        return PC_ERR_CUDA;
    int nfrozen = 0, j = 0;
    for (int i = 0; i < N; ++i) {
        if ((fz[i >> 5] >> (i & 31)) & 1u) {
            ++nfrozen;
            if (!da.empty() && ((da[i >> 5] >> (i & 31)) & 1u))
                return PC_ERR_INVALID; // a decision-aided position must carry information
        } else {
            if (j >= k || ip[j] != i)
                return PC_ERR_INVALID; // info_pos must list the non-frozen positions in order
            ++j;
        }
    }
    if (nfrozen != N - k || j != k)
        return PC_ERR_INVALID;
    code->first_info = ip[0];
    code->seal = seal_of(code);
    return PC_OK;
}

const char *pc_strerror(int code)
{
    switch (code) {
    case PC_OK: return "ok";
    case PC_ERR_INVALID: return "invalid argument";
    case PC_ERR_UNSUPPORTED: return "configuration not supported by the compiled kernels";
    case PC_ERR_CUDA: return "CUDA runtime error";
    case PC_ERR_NO_DEVICE: return "no sm_100 CUDA device";
    default: return "unknown error";
    }
}

int64_t pc_workspace_bytes(void) { return 256; }

int pc_device_count(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int good = 0;
    for (int d = 0; d < n; ++d) {
        int major = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) == cudaSuccess && major == 10)
            ++good;
    }
    return good;
}

int pc_bp_decode(const float *llr, int32_t B, const pc_code_t *code, const pc_bp_cfg_t *cfg, uint32_t *u_bits,
                 uint32_t *payload, float *soft_u, float *soft_x, int32_t *iters, uint8_t *converged,
                 uint64_t *t_done, void *stream)
{
    int rc = check_code(code);
    if (rc)
        return rc;
    if (cfg == nullptr || B < 0 || (B > 0 && (llr == nullptr || iters == nullptr || converged == nullptr)))
        return PC_ERR_INVALID;
    if (cfg->i_max < 1 || cfg->g_mode < 0 || cfg->g_mode > 3 || cfg->stop_mode < 0 || cfg->stop_mode > 2 ||
        cfg->kernel < 0 || cfg->kernel > 3 || !(cfg->llr_max > 0.0f))
        return PC_ERR_INVALID;
    if (cfg->stop_mode == 0 && (code->crc_width == 0 || code->crc_cols == nullptr))
        return PC_ERR_INVALID;
    BpArgs a;
    a.llr = llr;
    a.B = B;
    a.code = to_device_code(*code);
    a.i_max = cfg->i_max;
    a.stop_mode = cfg->stop_mode;
    a.llr_max = cfg->llr_max;
    a.u_bits = u_bits;
    a.payload = payload;
    a.soft_u = soft_u;
    a.soft_x = soft_x;
    a.iters = iters;
    a.conv = converged;
    a.t_done = t_done;
    a.work = cfg->work;
    return launch_bp_decode(a, cfg->g_mode, cfg->threads_per_frame, cfg->kernel, (cudaStream_t)stream);
}

int pc_bp_iterate(float *l_msgs, float *r_msgs, int32_t B, const pc_code_t *code, const pc_bp_cfg_t *cfg,
                  void *stream)
{
    int rc = check_code(code);
    if (rc)
        return rc;
    if (cfg == nullptr || B < 0 || (B > 0 && (l_msgs == nullptr || r_msgs == nullptr)) || cfg->g_mode < 0 ||
        cfg->g_mode > 3 || cfg->g_mode == 2 || !(cfg->llr_max > 0.0f))
        return PC_ERR_INVALID;
    return launch_bp_iterate(l_msgs, r_msgs, B, code->n, cfg->g_mode, cfg->llr_max, (cudaStream_t)stream);
}

int pc_compact(const uint8_t *converged, int32_t B, int32_t *queue, int32_t *count, void *workspace, void *stream)
{
    (void)workspace;
    if (B < 0 || count == nullptr || (B > 0 && (converged == nullptr || queue == nullptr)))
        return PC_ERR_INVALID;
    return launch_compact(converged, B, queue, count, (cudaStream_t)stream);
}

int pc_scl_decode(const float *llr, int32_t B, const int32_t *queue, const int32_t *count, const pc_code_t *code,
                  const pc_scl_cfg_t *cfg, uint32_t *u_bits, uint32_t *payload, float *metric, uint8_t *crc_ok,
                  uint8_t *sel_by_crc, uint64_t *t_done, void *workspace, void *stream)
{
    int rc = check_code(code);
    if (rc)
        return rc;
    if (cfg == nullptr || B < 0 || workspace == nullptr || (B > 0 && llr == nullptr))
        return PC_ERR_INVALID;
    const int Lreq = cfg->L;
    if (Lreq < 1 || Lreq > PC_MAX_LIST)
        return PC_ERR_UNSUPPORTED;
    int L = 1; // lanes per frame: the next power of two (K3 v3 keeps Lreq paths on them)
    while (L < Lreq)
        L <<= 1;
    if (code->crc_width > 0 && code->crc_cols == nullptr)
        return PC_ERR_INVALID;
    SclArgs a;
    a.llr = llr;
    a.B = B;
    a.queue = queue;
    a.count = count;
    a.code = to_device_code(*code);
    a.metric_exact = cfg->metric_exact;
    a.f_exact = cfg->f_exact;
    a.list_cap = Lreq;
    a.u_bits = u_bits;
    a.payload = payload;
    a.metric = metric;
    a.crc_ok = crc_ok;
    a.sel = sel_by_crc;
    a.t_done = t_done;
    a.work = reinterpret_cast<int32_t *>(workspace);
    a.tbg = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(workspace) + 256);
    if (cfg->kernel < 0 || cfg->kernel > 3)
        return PC_ERR_INVALID;
    // L = 1 (SC): one warp per frame (sc1.cu), bit-identical to K3 v3 at L = 1
    if (L == 1 && (cfg->kernel == 3 || (cfg->kernel == 0 && sc1_eligible(a))))
        return sc1_eligible(a) ? launch_sc1(a, (cudaStream_t)stream) : PC_ERR_UNSUPPORTED;
    if (cfg->kernel == 3)
        return PC_ERR_UNSUPPORTED;
    int nv = cfg->virtual_levels;
    if (cfg->kernel != 1 && scl3_eligible(a, L)) {
        if (nv < 0)
            nv = code->n >= 10 ? 3 : (code->n >= 8 ? 2 : 0); // measured best at N = 1024..4096
        const int rc3 = scl3_prepare(a, L, nv);
        if (rc3)
            return rc3;
        return launch_scl3(a, L, cfg->warps_per_cta, (cudaStream_t)stream);
    }
    if (cfg->kernel == 2 || L != Lreq) // (v2 takes power-of-two list sizes only)
        return PC_ERR_UNSUPPORTED;
    if (nv < 0)
        nv = code->n >= 12 ? 4 : (code->n >= 10 ? 3 : (code->n >= 8 ? 2 : 0));
    scl_prepare(a, nv);
    return launch_scl(a, L, cfg->warps_per_cta, (cudaStream_t)stream);
}

int64_t pc_scl_workspace_bytes(const pc_code_t *code, const pc_scl_cfg_t *cfg)
{
    if (check_shape(code) || cfg == nullptr || cfg->L < 1 || cfg->L > PC_MAX_LIST)
        return -1;
    int L = 1;
    while (L < cfg->L)
        L <<= 1;
    SclArgs a{};
    a.code = to_device_code(*code);
    a.B = 1;
    if (cfg->kernel != 1 && scl3_eligible(a, L)) {
        int nv = cfg->virtual_levels;
        if (nv < 0)
            nv = code->n >= 10 ? 3 : (code->n >= 8 ? 2 : 0);
        if (scl3_prepare(a, L, nv))
            return -1;
        return scl3_workspace_bytes(a, L, cfg->warps_per_cta);
    }
    return pc_workspace_bytes();
}

int pc_encode(const uint32_t *msg_bits, int32_t B, const pc_code_t *code, uint32_t *x_bits, void *stream)
{
    int rc = check_code(code);
    if (rc)
        return rc;
    if (B < 0 || (B > 0 && (msg_bits == nullptr || x_bits == nullptr)) ||
        (code->crc_width > 0 && code->enc_cols == nullptr))
        return PC_ERR_INVALID;
    return launch_encode(to_device_code(*code), msg_bits, B, x_bits, (cudaStream_t)stream);
}

int pc_gen_frames(uint64_t seed, int32_t point, int64_t frame0, int32_t B, float sigma, const pc_code_t *code,
                  uint32_t *msg_bits, float *llr, void *stream)
{
    int rc = check_code(code);
    if (rc)
        return rc;
    if (B < 0 || (B > 0 && llr == nullptr) || !(sigma >= 0.0f) || (code->crc_width > 0 && code->enc_cols == nullptr))
        return PC_ERR_INVALID;
    return launch_gen(to_device_code(*code), seed, point, frame0, B, sigma, msg_bits, llr, (cudaStream_t)stream);
}

int pc_count_errors(const uint32_t *payload, const uint32_t *msg_bits, int32_t B, int32_t m, int64_t *counters,
                    void *stream)
{
    if (B < 0 || m < 1 || counters == nullptr || (B > 0 && (payload == nullptr || msg_bits == nullptr)))
        return PC_ERR_INVALID;
    return launch_count_errors(payload, msg_bits, B, m, counters, (cudaStream_t)stream);
}

int pc_stamp(uint64_t *t, void *stream)
{
    if (t == nullptr)
        return PC_ERR_INVALID;
    return launch_stamp(t, (cudaStream_t)stream);
}

} // extern "C"
