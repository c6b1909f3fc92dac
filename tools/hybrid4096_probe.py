"""Hybrid BP->SCL at the paper's published configuration (N=4096, L=32, R=1/2;
34 Mbit/s maximum on a GTX 980 Ti): device throughput per
Eb/N0 point on one B200 (device Philox frames, resident in HBM).

    gpurun -- python tools/hybrid4096_probe.py
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

code = CodeConfig(4096, 2048, crc=16)
B = 32768
dc = nat.device_code(code)
lib = nat.load()
st = nat.stream_handle()
MW = (code.message_len + 31) // 32
msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
llr = torch.zeros((B, code.N), device="cuda")
dec = HybridDecoder(code, BpConfig(), SclConfig(32), capacity=B)
for p, eb in enumerate((1.5, 2.0, 2.5, 3.0, 3.5)):
    nat.check(lib.pc_gen_frames(7, p, 0, B, ebno_to_sigma(eb, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), st),
              "gen")
    dec.run(llr, B).sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        dec.run(llr, B)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    r = dec.host_results()
    gamma = float((~r["converged"]).mean())
    print(f"N=4096 L=32 {eb} dB: {B * code.message_len / ms / 1e6:.2f} Gbit/s ({ms:.1f} ms per {B} frames), "
          f"gamma={gamma:.4f}", flush=True)
