// torch_ops.cpp -- the C-ABI (include/polarcuda.h) exposed as a PyTorch
// extension: torch.classes.polar.Code and torch.ops.polar.{bp_decode,
// scl_decode, hybrid_decode, gen_frames, encode}.  Tensors in, tensors out,
// launches on the current CUDA stream; every op is a thin shim over one or
// three pc_* calls (no computation here).  Built by build_torch_ops.py
// against the installed torch; loaded with torch.ops.load_library
// (paper_1609_09358_b200/ops.py).
#include <ATen/ATen.h>
#include <c10/cuda/CUDAGuard.h>
#include <c10/cuda/CUDAStream.h>
#include <torch/custom_class.h>
#include <torch/library.h>

#include "polarcuda.h"

namespace {

void ok(int rc, const char *what)
{
    TORCH_CHECK(rc == PC_OK, what, ": ", pc_strerror(rc));
}

void *stream_of(const at::Tensor &t) { return c10::cuda::getCurrentCUDAStream(t.device().index()).stream(); }

void check_cuda(const at::Tensor &t, at::ScalarType dt, const char *name)
{
    TORCH_CHECK(t.is_cuda(), name, " must be a CUDA tensor");
    TORCH_CHECK(t.scalar_type() == dt, name, " has the wrong dtype");
    TORCH_CHECK(t.is_contiguous(), name, " must be contiguous");
}

// A code's device tables plus its sealed pc_code_t (CodeConfig, polar.py:216-286).
struct PolarCode : torch::CustomClassHolder {
    at::Tensor frozen_bits, crc_cols, info_pos, enc_cols, da_bits;
    pc_code_t c{};

    PolarCode(int64_t N, int64_t k, int64_t m, int64_t crc_width, int64_t crc_offset, int64_t enc_crc_offset,
              at::Tensor frozen_bits_, at::Tensor crc_cols_, at::Tensor info_pos_, at::Tensor enc_cols_,
              c10::optional<at::Tensor> da_bits_)
        : frozen_bits(std::move(frozen_bits_)), crc_cols(std::move(crc_cols_)), info_pos(std::move(info_pos_)),
          enc_cols(std::move(enc_cols_))
    {
        for (auto *t : {&frozen_bits, &crc_cols, &info_pos, &enc_cols})
            check_cuda(*t, at::kInt, "code table");
        int n = 0;
        while ((1LL << n) < N)
            ++n;
        c.N = (int32_t)N;
        c.n = n;
        c.k = (int32_t)k;
        c.m = (int32_t)m;
        c.crc_width = (int32_t)crc_width;
        c.crc_offset = (uint32_t)crc_offset;
        c.enc_crc_offset = (uint32_t)enc_crc_offset;
        c.first_info = 0; // derived by pc_code_seal
        c.frozen_bits = reinterpret_cast<const uint32_t *>(frozen_bits.data_ptr());
        c.crc_cols = reinterpret_cast<const uint32_t *>(crc_cols.data_ptr());
        c.info_pos = reinterpret_cast<const int32_t *>(info_pos.data_ptr());
        c.enc_cols = reinterpret_cast<const uint32_t *>(enc_cols.data_ptr());
        c.da_bits = nullptr;
        if (da_bits_.has_value()) {
            da_bits = *da_bits_;
            check_cuda(da_bits, at::kInt, "da_bits");
            c.da_bits = reinterpret_cast<const uint32_t *>(da_bits.data_ptr());
        }
        c10::cuda::CUDAGuard g(frozen_bits.device());
        ok(pc_code_seal(&c, stream_of(frozen_bits)), "pc_code_seal");
    }
    int64_t N() const { return c.N; }
    int64_t m() const { return c.m; }
};

using Code = c10::intrusive_ptr<PolarCode>;

at::Tensor empty_i32(const at::Tensor &like, std::initializer_list<int64_t> shape)
{
    return at::zeros(shape, like.options().dtype(at::kInt));
}

// bp_decode (bp.py:194-217) over a batch: iterations with the stop rule after each.
std::tuple<at::Tensor, at::Tensor, at::Tensor, at::Tensor, at::Tensor, at::Tensor>
bp_decode(const Code &code, const at::Tensor &llr, int64_t i_max, int64_t g_mode, int64_t stop_mode, double llr_max,
          bool soft)
{
    check_cuda(llr, at::kFloat, "llr");
    TORCH_CHECK(llr.dim() == 2 && llr.size(1) == code->c.N, "llr must be (B, N)");
    c10::cuda::CUDAGuard g(llr.device());
    const int64_t B = llr.size(0), N = code->c.N;
    auto u = empty_i32(llr, {B, (N + 31) / 32});
    auto pay = empty_i32(llr, {B, (code->c.m + 31) / 32});
    auto it = empty_i32(llr, {B});
    auto cv = at::zeros({B}, llr.options().dtype(at::kByte));
    at::Tensor su, sx;
    if (soft) {
        su = at::zeros({B, N}, llr.options());
        sx = at::zeros({B, N}, llr.options());
    }
    pc_bp_cfg_t cfg{};
    cfg.i_max = (int32_t)i_max;
    cfg.g_mode = (int32_t)g_mode;
    cfg.stop_mode = (int32_t)stop_mode;
    cfg.threads_per_frame = 0;
    cfg.llr_max = (float)llr_max;
    cfg.kernel = 0;
    cfg.work = nullptr;
    ok(pc_bp_decode(llr.data_ptr<float>(), (int32_t)B, &code->c, &cfg, reinterpret_cast<uint32_t *>(u.data_ptr()),
                    reinterpret_cast<uint32_t *>(pay.data_ptr()), soft ? su.data_ptr<float>() : nullptr,
                    soft ? sx.data_ptr<float>() : nullptr, it.data_ptr<int32_t>(), cv.data_ptr<uint8_t>(), nullptr,
                    stream_of(llr)),
       "pc_bp_decode");
    return {u, pay, it, cv, su, sx};
}

pc_scl_cfg_t scl_cfg(int64_t L, bool metric_exact, bool f_exact, bool bitonic)
{
    pc_scl_cfg_t s{};
    s.L = (int32_t)L;
    s.metric_exact = metric_exact;
    s.f_exact = f_exact;
    s.selector_bitonic = bitonic;
    s.virtual_levels = -1;
    s.warps_per_cta = 1;
    s.kernel = 0;
    return s;
}

at::Tensor workspace(const Code &code, const pc_scl_cfg_t &s, const at::Tensor &like)
{
    const int64_t bytes = pc_scl_workspace_bytes(&code->c, &s);
    TORCH_CHECK(bytes > 0, "pc_scl_workspace_bytes rejected the configuration");
    return at::empty({(bytes + 3) / 4}, like.options().dtype(at::kInt));
}

// scl_decode (scl.py:151-197) over a batch: CRC-aided list decoding, winner rule.
std::tuple<at::Tensor, at::Tensor, at::Tensor, at::Tensor, at::Tensor>
scl_decode(const Code &code, const at::Tensor &llr, int64_t L, bool metric_exact, bool f_exact, bool bitonic)
{
    check_cuda(llr, at::kFloat, "llr");
    TORCH_CHECK(llr.dim() == 2 && llr.size(1) == code->c.N, "llr must be (B, N)");
    c10::cuda::CUDAGuard g(llr.device());
    const int64_t B = llr.size(0), N = code->c.N;
    const pc_scl_cfg_t s = scl_cfg(L, metric_exact, f_exact, bitonic);
    auto ws = workspace(code, s, llr);
    auto u = empty_i32(llr, {B, (N + 31) / 32});
    auto pay = empty_i32(llr, {B, (code->c.m + 31) / 32});
    auto mt = at::zeros({B}, llr.options());
    auto okf = at::zeros({B}, llr.options().dtype(at::kByte));
    auto sel = at::zeros({B}, llr.options().dtype(at::kByte));
    ok(pc_scl_decode(llr.data_ptr<float>(), (int32_t)B, nullptr, nullptr, &code->c, &s,
                     reinterpret_cast<uint32_t *>(u.data_ptr()), reinterpret_cast<uint32_t *>(pay.data_ptr()),
                     mt.data_ptr<float>(), okf.data_ptr<uint8_t>(), sel.data_ptr<uint8_t>(), nullptr, ws.data_ptr(),
                     stream_of(llr)),
       "pc_scl_decode");
    return {u, pay, mt, okf, sel};
}

// hybrid_decode_batch (hybrid.py:153-258) on one stream: K1 (BP, CRC stop) ->
// K2 (queue of the failures) -> K3 (CRC-aided SCL from the original LLRs).
std::tuple<at::Tensor, at::Tensor, at::Tensor>
hybrid_decode(const Code &bp_code, const Code &scl_code, const at::Tensor &llr, int64_t i_max, double llr_max,
              int64_t L, bool metric_exact, bool f_exact)
{
    check_cuda(llr, at::kFloat, "llr");
    TORCH_CHECK(llr.dim() == 2 && llr.size(1) == bp_code->c.N && scl_code->c.N == bp_code->c.N,
                "llr must be (B, N)");
    c10::cuda::CUDAGuard g(llr.device());
    const int64_t B = llr.size(0);
    void *st = stream_of(llr);
    auto pay = empty_i32(llr, {B, (bp_code->c.m + 31) / 32});
    auto it = empty_i32(llr, {B});
    auto cv = at::zeros({B}, llr.options().dtype(at::kByte));
    auto queue = empty_i32(llr, {B > 0 ? B : 1});
    auto count = empty_i32(llr, {1});
    pc_bp_cfg_t cfg{};
    cfg.i_max = (int32_t)i_max;
    cfg.g_mode = 0;
    cfg.stop_mode = 0;
    cfg.llr_max = (float)llr_max;
    ok(pc_bp_decode(llr.data_ptr<float>(), (int32_t)B, &bp_code->c, &cfg, nullptr,
                    reinterpret_cast<uint32_t *>(pay.data_ptr()), nullptr, nullptr, it.data_ptr<int32_t>(),
                    cv.data_ptr<uint8_t>(), nullptr, st),
       "pc_bp_decode");
    ok(pc_compact(cv.data_ptr<uint8_t>(), (int32_t)B, queue.data_ptr<int32_t>(), count.data_ptr<int32_t>(), nullptr,
                  st),
       "pc_compact");
    const pc_scl_cfg_t s = scl_cfg(L, metric_exact, f_exact, false);
    auto ws = workspace(scl_code, s, llr);
    ok(pc_scl_decode(llr.data_ptr<float>(), (int32_t)B, queue.data_ptr<int32_t>(), count.data_ptr<int32_t>(),
                     &scl_code->c, &s, nullptr, reinterpret_cast<uint32_t *>(pay.data_ptr()), nullptr, nullptr,
                     nullptr, nullptr, ws.data_ptr(), st),
       "pc_scl_decode");
    return {pay, cv, it};
}

// Keyed synthetic frames (sim.py:117-121 semantics, Philox keys (seed, point, frame)).
std::tuple<at::Tensor, at::Tensor> gen_frames(const Code &code, int64_t seed, int64_t point, int64_t frame0,
                                              int64_t B, double sigma)
{
    const auto dev = code->frozen_bits.device();
    c10::cuda::CUDAGuard g(dev);
    auto opt = code->frozen_bits.options();
    auto msg = at::zeros({B, (code->c.m + 31) / 32}, opt.dtype(at::kInt));
    auto llr = at::zeros({B, (int64_t)code->c.N}, opt.dtype(at::kFloat));
    ok(pc_gen_frames((uint64_t)seed, (int32_t)point, frame0, (int32_t)B, (float)sigma, &code->c,
                     reinterpret_cast<uint32_t *>(msg.data_ptr()), llr.data_ptr<float>(), stream_of(llr)),
       "pc_gen_frames");
    return {msg, llr};
}

// polar_transform(insert_message(msg)) (polar.py:79-103) on bit-packed words.
at::Tensor encode(const Code &code, const at::Tensor &msg_bits)
{
    check_cuda(msg_bits, at::kInt, "msg_bits");
    c10::cuda::CUDAGuard g(msg_bits.device());
    const int64_t B = msg_bits.size(0);
    auto x = empty_i32(msg_bits, {B, ((int64_t)code->c.N + 31) / 32});
    ok(pc_encode(reinterpret_cast<const uint32_t *>(msg_bits.data_ptr()), (int32_t)B, &code->c,
                 reinterpret_cast<uint32_t *>(x.data_ptr()), stream_of(msg_bits)),
       "pc_encode");
    return x;
}

} // namespace

TORCH_LIBRARY(polar, m)
{
    m.class_<PolarCode>("Code")
        .def(torch::init<int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, at::Tensor, at::Tensor, at::Tensor,
                         at::Tensor, c10::optional<at::Tensor>>())
        .def("N", &PolarCode::N)
        .def("m", &PolarCode::m);
    m.def("bp_decode", bp_decode);
    m.def("scl_decode", scl_decode);
    m.def("hybrid_decode", hybrid_decode);
    m.def("gen_frames", gen_frames);
    m.def("encode", encode);
}
