"""Small launches of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck) — the race-detection leg of SURVEY.md's aux subsystems.

    compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_probe.py
    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1609_09358_b200 import (BpConfig, CodeConfig, HybridDecoder, SclConfig, bp_decode,  # noqa: E402
                                   bp_decode_batch, scl_decode_batch)
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def frames(N, eb, count, seed):
    code = CodeConfig(N, N // 2, crc=16)
    sigma = ebno_to_sigma(eb, code.rate)
    return code, np.array([make_frame(code, sigma, frame_rng(seed, N, f))[1] for f in range(count)])


for N in (64, 128, 256, 512, 1024, 2048, 4096):
    code, llrs = frames(N, 2.0, B, 1)
    for mode in ("crc", "reencode", "none"):
        bp_decode_batch(llrs, code, BpConfig(i_max=6, stop_mode=mode))  # k_bp3 (N >= 256), k_bp2, k_bp_decode
    bp_decode(llrs[0], code, BpConfig(i_max=4, stop_mode="crc"))
    bp_decode_batch(llrs, code, BpConfig(i_max=4, g_mode="min", stop_mode="crc"))
    for L in (1, 4, 32):  # L = 1: the SC kernel (one frame per warp at this batch size)
        scl_decode_batch(llrs, code, SclConfig(L))
    print("N", N, "ok", flush=True)

# the SC kernel's throughput form (G = 8 frames per warp: more than 8 frames per SM)
code, llrs = frames(256, 1.5, 1200, 3)
scl_decode_batch(llrs, code, SclConfig(1))
print("sc throughput form ok", flush=True)

code, llrs = frames(1024, 1.5, 4 * B, 2)
x = torch.from_numpy(llrs.astype(np.float32)).cuda()
dec = HybridDecoder(code, BpConfig(stop_mode="crc"), SclConfig(32))
dec.run(x)
dec.sync()
twin = HybridDecoder(code, BpConfig(stop_mode="crc"), SclConfig(32))
dec.run(x, join=False)  # cross-batch overlap: the twin's BP stage beside this SCL stage
twin.run(x, join=False)
dec.join_streams()
twin.join_streams()
torch.cuda.synchronize()
print("hybrid ok")
