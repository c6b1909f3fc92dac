#!/bin/bash
# K3 time per launch (L = 32 and 8, N = 1024 / 2048) for library variants (development aid)
for lib in "$@"; do
  cp "$lib" paper_1609_09358_b200/libpolarcuda.so
  echo "== $lib"
  timeout 300 python - <<'PY'
import ctypes, sys
sys.path.insert(0, ".")
import torch
from paper_1609_09358_b200 import CodeConfig, SclConfig
from paper_1609_09358_b200 import _native as nat
from paper_1609_09358_b200.channel import ebno_to_sigma
lib = nat.load()
for N, L, eb, B in ((1024, 32, 1.5, 32768), (1024, 32, 1.0, 32768), (2048, 8, 2.0, 32768), (2048, 32, 2.0, 16384), (4096, 32, 2.0, 8192), (1024, 4, 1.5, 32768)):
    code = CodeConfig(N, N // 2, crc=16); dc = nat.device_code(code)
    llr = torch.empty((B, N), device="cuda"); msg = torch.empty((B, N // 32), dtype=torch.int32, device="cuda")
    nat.check(lib.pc_gen_frames(3, 0, 0, B, ebno_to_sigma(eb, code.rate), dc.ref, msg.data_ptr(), llr.data_ptr(), nat.stream_handle()), "g")
    cfg = SclConfig(L).native(); ws = dc.new_scl_workspace(cfg)
    u = torch.zeros((B, N // 32), dtype=torch.int32, device="cuda"); mt = torch.zeros(B, device="cuda")
    run = lambda: nat.check(lib.pc_scl_decode(llr.data_ptr(), B, None, None, dc.ref, ctypes.byref(cfg), u.data_ptr(), None, mt.data_ptr(), None, None, None, ws.data_ptr(), nat.stream_handle()), "s")
    run(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [run() for _ in range(3)]; b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"N={N} L={L} {eb} dB: {B / ms / 1e3:.3f} Mframes/s  checksum {int(u.sum())} {float(mt.sum()):.3f}", flush=True)
PY
done
