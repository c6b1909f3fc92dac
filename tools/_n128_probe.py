import os, sys
sys.path.insert(0, ".")
import torch
from paper_1609_09358_b200 import BpConfig, CodeConfig, bp_decode_batch
from paper_1609_09358_b200 import _native as nat
from paper_1609_09358_b200.channel import ebno_to_sigma
N = int(sys.argv[1])
code = CodeConfig(N, N // 2, crc=16)
B = 1 << 16
dc = nat.device_code(code); lib = nat.load(); st = nat.stream_handle()
MW = (code.message_len + 31) // 32
msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
llr = torch.zeros((B, N), device="cuda")
nat.check(lib.pc_gen_frames(3, 0, 0, B, ebno_to_sigma(2.0, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), st), "g")
for k in ("2", "3"):
    os.environ["PC_BP_KERNEL"] = k
    r = bp_decode_batch(llr, code, BpConfig(stop_mode="crc"))
    torch.cuda.synchronize()
    print(k, r.iterations_used.to(torch.int64).sum().item() / B)
