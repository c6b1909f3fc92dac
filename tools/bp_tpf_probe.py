"""K1 time per launch for several threads-per-frame settings (development aid).

    python tools/bp_tpf_probe.py N ebno frames tpf1,tpf2,...
"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

N, EB, B = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
TPFS = [int(x) for x in sys.argv[4].split(",")]
code = CodeConfig(N, N // 2, crc=16)
dc = nat.device_code(code)
lib = nat.load()
st = nat.stream_handle()
MW = (code.message_len + 31) // 32
msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
llr = torch.zeros((B, N), device="cuda")
nat.check(lib.pc_gen_frames(5, 0, 0, B, ebno_to_sigma(EB, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), st), "g")
pay = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
ref = None
for tpf in TPFS:
    it = torch.zeros(B, dtype=torch.int32, device="cuda")
    cv = torch.zeros(B, dtype=torch.uint8, device="cuda")
    cfg = BpConfig(stop_mode="crc").native(threads_per_frame=tpf)

    def run():
        nat.check(lib.pc_bp_decode(llr.data_ptr(), B, dc.ref, ctypes.byref(cfg), None, pay.data_ptr(), None, None,
                                   it.data_ptr(), cv.data_ptr(), None, st), f"bp tpf={tpf}")

    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    g = int(it.to(torch.int64).sum()) * 2 * code.n * N
    same = ref is None or torch.equal(it, ref)
    ref = it.clone() if ref is None else ref
    print(f"N={N} tpf={tpf}: {ms:.2f} ms  {g / ms / 1e6:.1f} Gg/s  iterations identical: {same}", flush=True)
