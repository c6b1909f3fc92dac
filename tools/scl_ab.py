"""A/B of the SCL kernels (v2 per-leaf vs v3 register-block): identical
u_hat / metric / crc flags on the same frames, and batch throughput.

    python tools/scl_ab.py [N K L ebno frames]
"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import CodeConfig, SclConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
K = int(sys.argv[2]) if len(sys.argv) > 2 else N // 2
L = int(sys.argv[3]) if len(sys.argv) > 3 else 32
EB = float(sys.argv[4]) if len(sys.argv) > 4 else 1.5
B = int(sys.argv[5]) if len(sys.argv) > 5 else 8192

code = CodeConfig(N, K, crc=16)
dc = nat.device_code(code)
lib = nat.load()
st = nat.stream_handle()
MW = (code.message_len + 31) // 32
NW = (N + 31) // 32
msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
llr = torch.zeros((B, N), device="cuda")
nat.check(lib.pc_gen_frames(77, 0, 0, B, ebno_to_sigma(EB, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), st), "g")
out = {}
for kern in (1, 2):
    for nv in ((-1,) if kern == 1 else (-1, 2, 3, 4)):
        cfg = SclConfig(L).native(kernel=kern, virtual_levels=nv)
        u = torch.zeros((B, NW), dtype=torch.int32, device="cuda")
        pay = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
        mt = torch.zeros(B, device="cuda")
        ok = torch.zeros(B, dtype=torch.uint8, device="cuda")

        def run():
            nat.check(lib.pc_scl_decode(llr.data_ptr(), B, None, None, dc.ref, ctypes.byref(cfg), u.data_ptr(),
                                        pay.data_ptr(), mt.data_ptr(), ok.data_ptr(), None, None,
                                        dc.scl_workspace(cfg).data_ptr(), st), f"scl kernel={kern}")

        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        out[(kern, nv)] = (u.clone(), pay.clone(), mt.clone(), ok.clone())
        print(f"kernel v{kern + 1} nv={nv}: {ms:.2f} ms  {B / ms / 1e3:.3f} Mframes/s  "
              f"{B * code.message_len / ms / 1e6:.3f} Gbit/s", flush=True)
ref = out[(1, -1)]
for key, v in out.items():
    same = [torch.equal(x, y) for x, y in zip(ref, v)]
    bad = (ref[0] != v[0]).any(dim=1).nonzero().flatten().tolist()
    print(key, "u/pay/metric/ok identical:", same, "frames differing:", bad[:10], len(bad))
