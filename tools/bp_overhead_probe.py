"""Per-frame overhead of K1: frame-iterations/s with the CRC stop vs the
fixed cap (stop "none") at several i_max, same frames.

    gpurun -- python tools/bp_overhead_probe.py [N]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig, bp_decode_batch  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

for N in [int(a) for a in sys.argv[1:]] or [128, 1024, 4096]:
    code = CodeConfig(N, N // 2, crc=16)
    B = {128: 1 << 20, 1024: 65536}.get(N, 16384)
    dc = nat.device_code(code)
    lib = nat.load()
    st = nat.stream_handle()
    MW = (code.message_len + 31) // 32
    msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
    llr = torch.zeros((B, N), device="cuda")
    nat.check(lib.pc_gen_frames(3, 0, 0, B, ebno_to_sigma(2.0, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(),
                                st), "g")
    for mode, imax in (("crc", 50), ("none", 1), ("none", 2), ("none", 5), ("none", 10), ("none", 50)):
        cfg = BpConfig(stop_mode=mode, i_max=imax)
        r = bp_decode_batch(llr, code, cfg)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            r = bp_decode_batch(llr, code, cfg)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        its = r.iterations_used.to(torch.int64).sum().item()
        print(f"N={N} stop={mode} i_max={imax}: {ms:.2f} ms, {its / B:.2f} it/frame, "
              f"{its / ms / 1e3:.1f} M frame-it/s, {ms * 1e6 / B:.1f} ns/frame", flush=True)
