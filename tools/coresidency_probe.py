"""Upper bound of BP/SCL co-scheduling at the c3 1 dB point (development aid):
K1 over 131072 frames and K3 (L=32) over the 1 dB point's BP failures, each
alone and both at once on two streams (no queue between them: independent
inputs, the best case a persistent SCL consumer pulling from a device ring
could reach).

    python tools/coresidency_probe.py [ebno]
"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig, SclConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

EB = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
B, NS = 131072, 89255
code = CodeConfig(1024, 512, crc=16)
dc = nat.device_code(code)
lib = nat.load()
MW = (code.message_len + 31) // 32
msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
llr = torch.zeros((B, 1024), device="cuda")
nat.check(lib.pc_gen_frames(3, 0, 0, B, ebno_to_sigma(EB, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(),
                            nat.stream_handle()), "gen")
pay = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
pay2 = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
it = torch.zeros(B, dtype=torch.int32, device="cuda")
cv = torch.zeros(B, dtype=torch.uint8, device="cuda")
work = torch.zeros(1, dtype=torch.int32, device="cuda")
bcfg = BpConfig(i_max=50, stop_mode="crc").native()
bcfg.work = work.data_ptr()
scfg = SclConfig(32).native()
ws = dc.new_scl_workspace(scfg)
s1 = torch.cuda.Stream()
s2 = torch.cuda.Stream(priority=-1)  # the SCL stream's priority in HybridDecoder


def k1(s):
    nat.check(lib.pc_bp_decode(llr.data_ptr(), B, dc.ref, ctypes.byref(bcfg), None, pay.data_ptr(), None, None,
                               it.data_ptr(), cv.data_ptr(), None, ctypes.c_void_p(s.cuda_stream)), "bp")


def k3(s):
    nat.check(lib.pc_scl_decode(llr.data_ptr(), NS, None, None, dc.ref, ctypes.byref(scfg), None, pay2.data_ptr(),
                                None, None, None, None, ws.data_ptr(), ctypes.c_void_p(s.cuda_stream)), "scl")


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def both(first_k1):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    if first_k1:
        k1(s1)
        k3(s2)
    else:
        k3(s2)
        k1(s1)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1 = timed(lambda: k1(torch.cuda.current_stream()))
t3 = timed(lambda: k3(torch.cuda.current_stream()))
tb1 = timed(lambda: both(True))
tb3 = timed(lambda: both(False))
print(f"{EB} dB: K1 alone {t1:.2f} ms, K3 alone ({NS} frames) {t3:.2f} ms, sum {t1 + t3:.2f} ms; "
      f"together (K1 launched first) {tb1:.2f} ms = {tb1 / (t1 + t3):.3f} of the sum, "
      f"(K3 first) {tb3:.2f} ms = {tb3 / (t1 + t3):.3f}", flush=True)
