"""One launch of the SC kernel (sc1.cu) for ncu: N=2048 K=1024 CRC-16, 2 dB.
    args: [frames]"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import CodeConfig, SclConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
code = CodeConfig(2048, 1024, crc=16)
dc = nat.device_code(code)
lib = nat.load()
llr = torch.zeros((max(B, 1), 2048), device="cuda")
msg = torch.zeros((max(B, 1), 32), dtype=torch.int32, device="cuda")
nat.check(lib.pc_gen_frames(5, 0, 0, B, ebno_to_sigma(2.0, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(),
                            nat.stream_handle()), "gen")
ncfg = SclConfig(1).native(kernel=3)
ws = dc.new_scl_workspace(ncfg)
u = torch.zeros((B, 64), dtype=torch.int32, device="cuda")
nat.check(lib.pc_scl_decode(llr.data_ptr(), B, None, None, dc.ref, ctypes.byref(ncfg), u.data_ptr(), None, None,
                            None, None, None, ws.data_ptr(), nat.stream_handle()), "scl")
torch.cuda.synchronize()
print("sc1 frames", B)
