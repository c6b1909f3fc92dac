"""One launch each of K1 (BP) and K3 (SCL) on 2 dB frames, for ncu captures.
    args: [bp_frames scl_frames ebno N]

    ncu --set full --clock-control none --import-source on -k regex:k_bp_decode -c 1 \
        -o gpurun_out/bp python tools/profile_kernels.py
"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig, SclConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

B_BP = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
B_SCL = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
EB = float(sys.argv[3]) if len(sys.argv) > 3 else 2.0
NN = int(sys.argv[4]) if len(sys.argv) > 4 else 1024

code = CodeConfig(NN, NN // 2, crc=16)
dc = nat.device_code(code)
lib = nat.load()
st = nat.stream_handle()
MW = (code.message_len + 31) // 32
B = max(B_BP, B_SCL)
msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
llr = torch.zeros((B, NN), device="cuda")
nat.check(lib.pc_gen_frames(3, 0, 0, B, ebno_to_sigma(EB, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), st), "g")
pay = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
it = torch.zeros(B, dtype=torch.int32, device="cuda")
cv = torch.zeros(B, dtype=torch.uint8, device="cuda")
cfg = BpConfig(stop_mode="crc").native()
work = torch.empty(1, dtype=torch.int32, device="cuda")  # frame counter: the persistent K1 at small N
cfg.work = work.data_ptr()
nat.check(lib.pc_bp_decode(llr.data_ptr(), B_BP, dc.ref, ctypes.byref(cfg), None, pay.data_ptr(), None, None,
                           it.data_ptr(), cv.data_ptr(), None, st), "bp")
scfg = SclConfig(32).native()
nat.check(lib.pc_scl_decode(llr.data_ptr(), B_SCL, None, None, dc.ref, ctypes.byref(scfg), None, pay.data_ptr(),
                            None, None, None, None, dc.scl_workspace(scfg).data_ptr(), st), "scl")
torch.cuda.synchronize()
print("bp frames", B_BP, "iterations", int(it[:B_BP].sum().item()), "scl frames", B_SCL)
