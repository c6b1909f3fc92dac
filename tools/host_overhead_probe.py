import sys, time
sys.path.insert(0, ".")
import torch
from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig
from paper_1609_09358_b200 import _native as nat
from paper_1609_09358_b200.channel import ebno_to_sigma
code = CodeConfig(1024, 512, crc=16); dc = nat.device_code(code); lib = nat.load()
NF = 4096
llr = torch.empty((NF, 1024), device="cuda"); msg = torch.empty((NF, 16), dtype=torch.int32, device="cuda")
nat.check(lib.pc_gen_frames(9, 0, 0, NF, ebno_to_sigma(2.0, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), nat.stream_handle()), "g")
for ch in (32, 1024):
    d = HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=NF, chunk=ch)
    d.run(llr).sync()
    t0 = time.perf_counter(); d.run(llr); t1 = time.perf_counter(); d.sync(); t2 = time.perf_counter()
    print(f"chunk {ch}: enqueue {1e3*(t1-t0):.2f} ms ({1e6*(t1-t0)/(NF//ch):.1f} us/chunk), total {1e3*(t2-t0):.2f} ms")
for ch in (32, 1024):
    d = HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=NF, chunk=ch)
    d.run(llr).sync()
    ref = d.host_results()
    d.run(llr, graph=True).sync()
    d.payload.zero_()
    d.conv.zero_()
    t0 = time.perf_counter(); d.run(llr, graph=True); t1 = time.perf_counter(); d.sync(); t2 = time.perf_counter()
    r = d.host_results()
    import numpy as np
    same = all(np.array_equal(r[k], ref[k]) for k in ("payload", "converged", "iters"))
    print(f"graph chunk {ch}: enqueue {1e3*(t1-t0):.2f} ms, total {1e3*(t2-t0):.2f} ms, same results {same}")
