"""K1 v3 (bp3.cu, layout transposes) against K1 v2 (bp2.cu, lane-pair
shuffles) at the same 8 nodes per thread: bit-identical iterations, flags,
decisions and soft outputs for every stop rule, and the time per launch.

    python tools/bp_kernel_ab.py [frames] [ebno]
"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1609_09358_b200 import BpConfig, CodeConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma  # noqa: E402

B0 = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
EB = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
lib = nat.load()
st = nat.stream_handle()
ok_all = True
for N in (256, 512, 1024, 2048, 4096):
    B = max(1024, B0 * 1024 // N)
    code = CodeConfig(N, N // 2, crc=16)
    dc = nat.device_code(code)
    MW = (code.message_len + 31) // 32
    msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
    llr = torch.zeros((B, N), device="cuda")
    nat.check(lib.pc_gen_frames(11, 0, 0, B, ebno_to_sigma(EB, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(),
                                st), "gen")
    work = torch.zeros(1, dtype=torch.int32, device="cuda")
    for g_mode in ("exact", "min"):
        for stop in ("crc", "reencode", "none"):
            if stop == "reencode" and N < 512:
                continue
            outs, times = [], []
            for kern in (2, 3):
                cfg = BpConfig(g_mode=g_mode, stop_mode=stop, i_max=50 if stop != "none" else 8).native(
                    threads_per_frame=N // 8, kernel=kern)
                cfg.work = work.data_ptr()
                Bs = B if stop == "crc" else min(B, 4096)
                pay = torch.zeros((Bs, MW), dtype=torch.int32, device="cuda")
                it = torch.zeros(Bs, dtype=torch.int32, device="cuda")
                cv = torch.zeros(Bs, dtype=torch.uint8, device="cuda")
                su = torch.zeros((Bs, N), device="cuda")
                sx = torch.zeros((Bs, N), device="cuda")

                def run(soft):
                    nat.check(lib.pc_bp_decode(llr.data_ptr(), Bs, dc.ref, ctypes.byref(cfg), None, pay.data_ptr(),
                                               su.data_ptr() if soft else None, sx.data_ptr() if soft else None,
                                               it.data_ptr(), cv.data_ptr(), None, st), f"bp k{kern}")

                run(True)
                torch.cuda.synchronize()
                outs.append([t.clone() for t in (pay, it, cv, su, sx)])
                ms = 0.0
                if stop == "crc":
                    run(False)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(3):
                        run(False)
                    b.record()
                    torch.cuda.synchronize()
                    ms = a.elapsed_time(b) / 3
                times.append(ms)
            same = [bool(torch.equal(x, y)) for x, y in zip(*outs)]
            ok_all &= all(same)
            g = int(outs[0][1].to(torch.int64).sum()) * 2 * code.n * N
            extra = ""
            if stop == "crc":
                extra = (f" v2 {times[0]:.3f} ms ({g / times[0] / 1e6:.0f} Gg/s)  v3 {times[1]:.3f} ms "
                         f"({g / times[1] / 1e6:.0f} Gg/s)  x{times[0] / times[1]:.3f}")
            print(f"N={N} {g_mode} {stop}: identical payload/iters/conv/soft_u/soft_x {same}{extra}", flush=True)
print("ALL_IDENTICAL" if ok_all else "DIFFERENCES")
