"""Re-encode stop vs CRC stop, and the two BP kernels (PC_BP_KERNEL=1/2), in
frame-iterations per second on 2.5 dB frames (K1 stop rule).

    gpurun -- python tools/reencode_probe.py
"""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1609_09358_b200 import BpConfig, CodeConfig, bp_decode_batch
from paper_1609_09358_b200 import _native as nat
from paper_1609_09358_b200.channel import ebno_to_sigma
for N in (1024, 4096):
    code = CodeConfig(N, N // 2, crc=16)
    B = 65536 if N == 1024 else 16384
    dc = nat.device_code(code); lib = nat.load(); st = nat.stream_handle()
    MW = (code.message_len + 31) // 32
    msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
    llr = torch.zeros((B, N), device="cuda")
    nat.check(lib.pc_gen_frames(3, 0, 0, B, ebno_to_sigma(2.5, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), st), "g")
    for mode in ("crc", "reencode"):
        for k in (("1", "2") if N == 1024 else ("2",)):
            os.environ["PC_BP_KERNEL"] = k
            r = bp_decode_batch(llr, code, BpConfig(stop_mode=mode))
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(3):
                r = bp_decode_batch(llr, code, BpConfig(stop_mode=mode))
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t) / 3
            its = r.iterations_used.sum().item()
            print(N, mode, "kernel", k, f"{dt*1e3:.2f} ms", f"{its/dt/1e6:.1f} M frame-iters/s", f"conv {r.converged.float().mean().item():.3f} avg_it {its/B:.2f}")
