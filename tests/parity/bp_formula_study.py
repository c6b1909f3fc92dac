"""Decision parity of the two exact-g evaluations against the fp64 oracle:
g_mode 0 (exponential domain, 3.5 MUFU/g) and g_mode 2 (per-g form, 4 MUFU/g).

For each set: frames whose converged flag or iteration count differ from the
oracle, split at the reference's iteration 20, and frames where both converged
but u_hat differs.  Writes a JSON summary.

    python tests/parity/bp_formula_study.py out.json
"""
import ctypes
import json
import sys

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1609_09358_b200 import BpConfig, CodeConfig  # noqa: E402
from paper_1609_09358_b200 import _native as nat  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame  # noqa: E402

SETS = [(1024, 1.5, 3000), (1024, 2.0, 3000), (1024, 2.5, 3000), (2048, 2.0, 1000)]
out = {}
lib = nat.load()
for N, eb, count in SETS:
    code = CodeConfig(N, N // 2, crc=16)
    sigma = ebno_to_sigma(eb, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(9090, int(10 * eb), f))[1] for f in range(count)])
    llrs = llrs.astype(np.float32).astype(np.float64)
    ref_u, ref_it, ref_cv = oracle.bp_batch(llrs, code, stop_mode="crc")
    x = torch.from_numpy(llrs.astype(np.float32)).cuda()
    dc = nat.device_code(code)
    NW = N // 32
    row = {}
    for gm in (0, 2):
        cfg = BpConfig(stop_mode="crc").native()
        cfg.g_mode = gm
        u = torch.zeros((count, NW), dtype=torch.int32, device="cuda")
        it = torch.zeros(count, dtype=torch.int32, device="cuda")
        cv = torch.zeros(count, dtype=torch.uint8, device="cuda")
        nat.check(lib.pc_bp_decode(x.data_ptr(), count, dc.ref, ctypes.byref(cfg), u.data_ptr(), None, None, None,
                                   it.data_ptr(), cv.data_ptr(), None, nat.stream_handle()), "bp")
        uh = nat.unpack_bits(u.cpu().numpy().view(np.uint32), N)
        it, cv = it.cpu().numpy(), cv.cpu().numpy().astype(bool)
        flag_or_iter = (cv != ref_cv.astype(bool)) | (it != ref_it)
        both = cv & ref_cv.astype(bool)
        u_diff = both & (uh != ref_u).any(axis=1)
        row[f"g_mode{gm}"] = {
            "early_flips": int((flag_or_iter & (ref_it <= 20)).sum()),
            "late_flips": int((flag_or_iter & (ref_it > 20)).sum()),
            "uhat_diff_both_converged": int(u_diff.sum()),
            "converged_flag_diff": int((cv != ref_cv.astype(bool)).sum()),
            "early_frames": [(int(f), int(ref_it[f]), int(it[f])) for f in np.flatnonzero(flag_or_iter & (ref_it <= 20))][:20],
        }
    out[f"N{N}_{eb}dB_{count}"] = row
    print(f"N{N} {eb} dB {count}:", json.dumps(row), flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "bp_formula_study.json", "w"), indent=1)
