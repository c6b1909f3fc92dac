"""Selection statistics of K3 at L = 32 (development aid; needs a library built
with -DSCL3_STATS, e.g. build/variants/stats.so copied over libpolarcuda.so):
share of full-list info leaves with an uncertain set, settled by one swap,
and with clones, on hybrid queues (BP failures) and on all frames.

    python tools/scl3_stats.py
"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig, scl_decode_batch  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

lib = nat.load()
lib.pc_debug_scl3_stats.argtypes = [ctypes.c_void_p]
code = CodeConfig(1024, 512, crc=16)
dc = nat.device_code(code)
out = (ctypes.c_ulonglong * 8)()
B = 16384
for eb in (1.0, 1.5, 2.0, 3.0):
    llr = torch.empty((B, 1024), device="cuda")
    msg = torch.empty((B, 16), dtype=torch.int32, device="cuda")
    nat.check(lib.pc_gen_frames(9, 0, 0, B, ebno_to_sigma(eb, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(),
                                nat.stream_handle()), "gen")
    for what in ("hybrid queue", "all frames"):
        lib.pc_debug_scl3_stats(out)
        if what == "hybrid queue":
            dec = HybridDecoder(code, BpConfig(), SclConfig(32), capacity=B)
            dec.run(llr).sync()
            nq = int((~dec.host_results()["converged"]).sum())
        else:
            scl_decode_batch(llr, code, SclConfig(32))
            nq = B
        torch.cuda.synchronize()
        lib.pc_debug_scl3_stats(out)
        full, unc, swap, clone = out[0], out[1], out[2], out[3]
        print(f"{eb} dB {what}: frames {nq}, full-list selections per frame {full / max(nq, 1):.0f}, "
              f"uncertain {unc / max(full, 1):.3f} (one swap {swap / max(full, 1):.3f}), "
              f"clones {clone / max(full, 1):.3f}", flush=True)
