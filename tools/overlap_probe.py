"""Sequential per-point hybrid runs vs one pipelined run over all Eb/N0
points (chunk c+1's BP overlapping chunk c's SCL on the two streams)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

EB = (1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
code = CodeConfig(1024, 512, crc=16)
lib = nat.load()
dc = nat.device_code(code)
MW = (code.message_len + 31) // 32
llr = torch.empty((len(EB) * B, 1024), device="cuda")
msg = torch.empty((len(EB) * B, MW), dtype=torch.int32, device="cuda")
for p, eb in enumerate(EB):
    nat.check(lib.pc_gen_frames(1, p, 0, B, ebno_to_sigma(eb, code.rate), dc.ref, msg[p * B].data_ptr(),
                                llr[p * B].data_ptr(), nat.stream_handle()), "gen")


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


dec = HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=B, chunk=B)
seq = timeit(lambda: [dec.run(llr[p * B:(p + 1) * B], B) for p in range(len(EB))])
print(f"sequential per point: {seq:.1f} ms  {len(EB) * B * 496 / seq / 1e6:.3f} Gbit/s", flush=True)
for div in (1, 2, 4, 8):
    big = HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=len(EB) * B, chunk=B // div)
    t = timeit(lambda: big.run(llr, len(EB) * B))
    print(f"pipelined chunk=B/{div}: {t:.1f} ms  {len(EB) * B * 496 / t / 1e6:.3f} Gbit/s", flush=True)
    del big
