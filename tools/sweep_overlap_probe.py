"""Cross-point overlap of the hybrid pipeline (development aid): the c3 sweep
(7 points x B frames) run (a) point after point on one decoder (the BP stage
of point p+1 waits for the SCL stage of point p) and (b) on D ping-pong
decoders with run(join=False), so the BP stage of point p+1 overlaps the SCL
stage of point p.  Device time per sweep and the identical-results check.

    python tools/sweep_overlap_probe.py [B] [D] [chunk]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
D = int(sys.argv[2]) if len(sys.argv) > 2 else 2
CH = int(sys.argv[3]) if len(sys.argv) > 3 else B
EB = (1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0)
code = CodeConfig(1024, 512, crc=16)
dc = nat.device_code(code)
lib = nat.load()
MW = (code.message_len + 31) // 32
llr = torch.empty((len(EB), B, 1024), device="cuda")
msg = torch.empty((len(EB), B, MW), dtype=torch.int32, device="cuda")
for p, eb in enumerate(EB):
    nat.check(lib.pc_gen_frames(20240917, p, 0, B, ebno_to_sigma(eb, code.rate), dc.ref, msg[p].data_ptr(),
                                llr[p].data_ptr(), nat.stream_handle()), "gen")
decs = [HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=B, chunk=CH) for _ in range(D)]


def seq():
    for p in range(len(EB)):
        decs[0].run(llr[p], B)


def pingpong():
    for p in range(len(EB)):
        decs[p % D].run(llr[p], B, join=False)
    for d in decs:
        d.join_streams()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


bits = len(EB) * B * code.message_len
t1 = timed(seq)
t2 = timed(pingpong)
print(f"B={B} chunk={CH} D={D}: sequential {t1:.1f} ms ({bits / t1 / 1e6:.3f} Gbit/s), "
      f"ping-pong {t2:.1f} ms ({bits / t2 / 1e6:.3f} Gbit/s), gain {t1 / t2:.3f}x", flush=True)
# identical results: the last point decoded both ways
decs[0].run(llr[len(EB) - 1], B).sync()
ref = decs[0].payload[:B].clone()
pingpong()
torch.cuda.synchronize()
last = decs[(len(EB) - 1) % D]
print("last point payload identical:", bool(torch.equal(ref, last.payload[:B])))
