"""K1 time per launch for the exact-g arithmetic forms (development aid):
g_mode 0 (likelihood-ratio domain) vs 3 (round-1 exponential/log2 domain),
same device frames, several threads-per-frame settings.

    python tools/bp_gmode_probe.py N ebno frames tpf1,tpf2,... [gmodes=0,3]
"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

N, EB, B = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
TPFS = [int(x) for x in sys.argv[4].split(",")]
GMODES = [int(x) for x in (sys.argv[5] if len(sys.argv) > 5 else "0,3").split(",")]
code = CodeConfig(N, N // 2, crc=16)
dc = nat.device_code(code)
lib = nat.load()
st = nat.stream_handle()
MW = (code.message_len + 31) // 32
msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
llr = torch.zeros((B, N), device="cuda")
nat.check(lib.pc_gen_frames(5, 0, 0, B, ebno_to_sigma(EB, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), st), "g")
work = torch.zeros(1, dtype=torch.int32, device="cuda")
ref = None
for gm in GMODES:
    for tpf in TPFS:
        pay = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
        it = torch.zeros(B, dtype=torch.int32, device="cuda")
        cv = torch.zeros(B, dtype=torch.uint8, device="cuda")
        cfg = BpConfig(stop_mode="crc").native(threads_per_frame=tpf)
        cfg.g_mode = gm
        cfg.work = work.data_ptr()

        def run():
            nat.check(lib.pc_bp_decode(llr.data_ptr(), B, dc.ref, ctypes.byref(cfg), None, pay.data_ptr(), None,
                                       None, it.data_ptr(), cv.data_ptr(), None, st), f"bp g={gm} tpf={tpf}")

        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        g = int(it.to(torch.int64).sum()) * 2 * code.n * N
        errs = int(((pay != msg).any(dim=1)).sum())
        if ref is None:
            ref = (it.clone(), pay.clone())
        same_it = float((it == ref[0]).float().mean())
        same_pay = float(((pay == ref[1]).all(dim=1)).float().mean())
        print(f"N={N} {EB} dB g_mode={gm} tpf={tpf}: {ms:.3f} ms  {g / ms / 1e6:.1f} Gg/s  mean it "
              f"{float(it.float().mean()):.3f}  FER {errs / B:.5f}  BP-fail {1 - float(cv.float().mean()):.5f}  "
              f"same it/payload as first row {same_it:.5f}/{same_pay:.5f}", flush=True)
