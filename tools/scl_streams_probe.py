"""Hybrid pipeline at small chunks with 1..8 SCL streams (development aid):
wall throughput and p50 / p99 latency (batch start -> decision, the
reference's semantic) at chunk 32 and 1024, N=1024 L=32, 4096 frames.

    python tools/scl_streams_probe.py
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

code = CodeConfig(1024, 512, crc=16)
dc = nat.device_code(code)
lib = nat.load()
NF = 4096
MW = (code.message_len + 31) // 32
for eb in (1.0, 2.0):
    llr = torch.empty((NF, 1024), device="cuda")
    msg = torch.empty((NF, MW), dtype=torch.int32, device="cuda")
    nat.check(lib.pc_gen_frames(9, 0, 0, NF, ebno_to_sigma(eb, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(),
                                nat.stream_handle()), "gen")
    ref = None
    for ch in (32, 1024):
        for S in (1, 2, 4, 8):
            d = HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=NF, chunk=ch, scl_streams=S)
            d.run(llr).sync()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d.run(llr).sync()
            wall = time.perf_counter() - t0
            r = d.host_results()
            pay = r["payload"].copy()
            same = ref is None or np.array_equal(pay, ref)
            ref = pay if ref is None else ref
            st = r["stamps"]
            c = np.arange(NF) // ch
            done = np.where(r["converged"], r["t_bp"], r["t_scl"])
            lat = (done - st[c, 0]) * 1e-6
            print(f"{eb} dB chunk {ch} streams {S}: {NF * code.message_len / wall / 1e9:.3f} Gbit/s wall, "
                  f"p50 {np.median(lat):.3f} ms p99 {np.percentile(lat, 99):.3f} ms, payload same {same}", flush=True)
