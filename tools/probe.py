"""Quick device timing probe (development aid): BP, SCL, hybrid at N=1024.

    python tools/probe.py [B] [sections: bp,scl,hyb]
"""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

code = CodeConfig(1024, 512, crc=16)
dc = nat.device_code(code)
lib = nat.load()
st = nat.stream_handle()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
sections = sys.argv[2].split(",") if len(sys.argv) > 2 else ["bp", "scl", "hyb"]
MW = (code.message_len + 31) // 32
msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
llr = torch.zeros((B, 1024), device="cuda")
it = torch.zeros(B, dtype=torch.int32, device="cuda")
cv = torch.zeros(B, dtype=torch.uint8, device="cuda")
pay = torch.zeros((B, MW), dtype=torch.int32, device="cuda")


def ev():
    return torch.cuda.Event(enable_timing=True)


def gen(eb):
    nat.check(lib.pc_gen_frames(1, 0, 0, B, ebno_to_sigma(eb, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), st),
              "gen")


if "bp" in sections:
    for eb in (1.0, 2.0, 3.0, 4.0):
        gen(eb)
        for kern, tpf in ((1, 512), (2, 128), (2, 256), (2, 512)):
            cfg = BpConfig(stop_mode="crc").native(threads_per_frame=tpf, kernel=kern)
            for rep in range(2):
                a, b = ev(), ev()
                a.record()
                nat.check(lib.pc_bp_decode(llr.data_ptr(), B, dc.ref, ctypes.byref(cfg), None, pay.data_ptr(), None,
                                           None, it.data_ptr(), cv.data_ptr(), None, st), "bp")
                b.record()
                torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            iters = it.sum().item()
            gps = iters * 2 * 10 * 1024 / (ms * 1e-3)
            print(f"BP eb={eb} k={kern} tpf={tpf}: {ms:.2f} ms  mean_it={iters / B:.2f} "
                  f"gamma={(cv == 0).float().mean().item():.3f} g/s={gps:.3e} frac_xu(1.163e12)={gps / 1.163e12:.3f} "
                  f"info Gbit/s={B * 496 / (ms * 1e-3) / 1e9:.3f}")

if "scl" in sections:
    gen(1.5)
    for L in (1, 4, 8, 32):
        Bs = min(B, 8192 if L == 32 else 32768)
        for nv in (2, 3, 4):
            cfg = SclConfig(L).native(virtual_levels=nv, warps_per_cta=1)
            for rep in range(2):
                a, b = ev(), ev()
                a.record()
                nat.check(lib.pc_scl_decode(llr.data_ptr(), Bs, None, None, dc.ref, ctypes.byref(cfg), None,
                                            pay.data_ptr(), None, None, None, None, dc.scl_workspace(cfg).data_ptr(), st), "scl")
                b.record()
                torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            print(f"SCL L={L} nv={nv}: {ms:.2f} ms for {Bs} frames -> {Bs / (ms * 1e-3):.0f} frames/s, "
                  f"{Bs * 496 / (ms * 1e-3) / 1e9:.3f} Gbit/s")

if "hyb" in sections:
    for eb in (1.0, 1.5, 2.0, 3.0, 4.0):
        gen(eb)
        for chunk, overlap in ((B, True), (B // 4, True), (B // 8, True), (B // 16, True), (B // 8, False)):
            dec = HybridDecoder(code, BpConfig(), SclConfig(32), capacity=B, chunk=chunk, overlap=overlap)
            for rep in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                dec.run(llr).sync()
                t = time.perf_counter() - t0
            r = dec.host_results()
            print(f"HYB eb={eb} chunk={chunk} overlap={overlap}: {t * 1e3:.1f} ms gamma={(~r['converged']).mean():.4f} "
                  f"info Gbit/s={B * 496 / t / 1e9:.3f}")
