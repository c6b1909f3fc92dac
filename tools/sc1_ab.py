"""The one-warp-per-frame SC kernel (sc1.cu, pc_scl_cfg_t.kernel 3) against
K3 v3 at L = 1 (kernel 2): bit-identical u_hat, metric and CRC flags over
codes and knobs, then throughput (L = 1 vs L = 2) and single-frame latency
at N = 2048 (BASELINE configs[4]).

    python tools/sc1_ab.py
"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import CodeConfig, SclConfig, scl_decode_batch  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

lib = nat.load()


def frames(code, eb, B, seed=21):
    MW = (code.message_len + 31) // 32
    msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
    llr = torch.zeros((B, code.N), device="cuda")
    nat.check(lib.pc_gen_frames(seed, 0, 0, B, ebno_to_sigma(eb, code.rate), nat.device_code(code).ref,
                                msg.data_ptr(), llr.data_ptr(), nat.stream_handle()), "gen")
    return llr


def dec(llr, code, cfg, kernel):
    os.environ["PC_SCL_KERNEL"] = str(kernel)
    r = scl_decode_batch(llr, code, cfg, payload=True)
    torch.cuda.synchronize()
    return r


ok_all = True
for N, crc in ((64, 8), (128, 16), (256, None), (1024, 16), (2048, 16), (4096, 24)):
    code = CodeConfig(N, N // 2, crc=crc)
    llr = frames(code, 1.5, 1500)
    for fm, mm, da in (("minsum", "exact", 0.0), ("exact", "exact", 0.0), ("minsum", "approx", 0.0),
                       ("minsum", "exact", 0.3)):
        cfg = SclConfig(1, metric_mode=mm, f_mode=fm, da_threshold=da)
        a, b = dec(llr, code, cfg, 2), dec(llr, code, cfg, 3)
        same = [bool(torch.equal(x, y)) for x, y in ((a.u_hat, b.u_hat), (a.metric, b.metric),
                                                     (a.crc_ok, b.crc_ok), (a.payload_words, b.payload_words))]
        ok_all &= all(same)
        print(f"N={N} crc={crc} f={fm} metric={mm} da={da}: identical u/metric/crc/payload {same}", flush=True)
print("ALL_IDENTICAL" if ok_all else "DIFFERENCES", flush=True)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


code = CodeConfig(2048, 1024, crc=16)
llr = frames(code, 2.0, 32768, seed=5)
dc = nat.device_code(code)
B = 32768
u = torch.zeros((B, 64), dtype=torch.int32, device="cuda")
mt = torch.zeros(B, device="cuda")
import ctypes  # noqa: E402

for L, kern in ((1, 2), (1, 3), (2, 0), (4, 0), (32, 0)):
    ncfg = SclConfig(L).native(kernel=kern)
    ws = dc.new_scl_workspace(ncfg)

    def run(nb):
        nat.check(lib.pc_scl_decode(llr.data_ptr(), nb, None, None, dc.ref, ctypes.byref(ncfg), u.data_ptr(), None,
                                    mt.data_ptr(), None, None, None, ws.data_ptr(), nat.stream_handle()), "scl")

    ms = timed(lambda: run(B), 3)
    lat = timed(lambda: run(1), 50)
    print(f"N=2048 L={L} kernel={kern}: {B / ms / 1e3:.2f} Mframes/s, single frame {lat * 1e3:.1f} us "
          "(one frame alone on the GPU, CUDA events around the launch)", flush=True)
