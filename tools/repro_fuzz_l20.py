import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests/parity")
import numpy as np
import oracle
from paper_1609_09358_b200 import CodeConfig, SclConfig, scl_decode_batch
from fuzz_parity import frames
code = CodeConfig(4096, 1741, crc=None)
llrs = frames(code, -0.5708736772407244, 2, 100425)
for L in (20, 16, 24, 32, 17, 31):
    got = scl_decode_batch(llrs, code, SclConfig(L))
    bad = []
    for f in range(2):
        ref = oracle.scl_decode(llrs[f], code, L)
        if not np.array_equal(got.u_hat[f], ref["u_hat"]):
            bad.append((f, float(got.metric[f]), ref["metric"]))
    print("L", L, "bad", bad, flush=True)
# more random frames at N=4096 L=20, low SNR
for N, k, L, eb in ((4096, 1741, 20, -0.5), (2048, 900, 20, -0.5), (1024, 400, 20, -0.5), (4096, 1741, 12, 0.0), (4096, 2048, 24, 0.5)):
    code = CodeConfig(N, k, crc=None)
    llrs = frames(code, eb, 12, 777)
    got = scl_decode_batch(llrs, code, SclConfig(L))
    nb = sum(not np.array_equal(got.u_hat[f], oracle.scl_decode(llrs[f], code, L)["u_hat"]) for f in range(12))
    print(N, k, L, eb, "differing", nb, "of 12", flush=True)
