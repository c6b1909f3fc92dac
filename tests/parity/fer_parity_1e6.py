"""High-SNR FER parity with power: 10^6 paired frames per
point at 3.0 / 3.5 / 4.0 dB, device hybrid decoder vs the fp64 oracle port,
with Clopper-Pearson intervals on both sides and the paired sign test
(reference test_acceptance.py:55-61, 223-257).  The CRC-16 false-accept floor
of the reference algorithm (a wrong BP estimate that passes the per-iteration
CRC check) is visible on both sides.

Two phases, so the slow side does not hold the GPU:
    # on the B200: decode the keyed host frames, save per-frame error counts
    python tests/parity/fer_parity_1e6.py device gpurun_out/fer1e6_device.npz
    # anywhere with cores: the oracle on the same frames (regenerated), compare
    python tests/parity/fer_parity_1e6.py oracle gpurun_out/fer1e6_device.npz profiles/fer_parity_1e6.json
Options (both phases alike): --ebno 3,3.5,4 --frames 1000000 --point0 10, e.g. the
full sweep at 2 x 10^4 paired frames per point:
    ... device gpurun_out/fer20k_device.npz --ebno 1,1.5,2,2.5,3,3.5,4 --frames 20000 --point0 20
"""

from __future__ import annotations

import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

from fer_parity import IMAX, K, L, N, clopper_pearson, cluster_ci, host_frames  # noqa: E402

EBNO = (3.0, 3.5, 4.0)
FRAMES = 1_000_000
CHUNK = 65536
POINT0 = 10  # point keys 10, 11, 12: frames disjoint from fer_parity.py's


def device_phase(out):
    import torch

    import oracle
    from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig
    from paper_1609_09358_b200 import _native as nat

    code = CodeConfig(N, K, crc=16)
    m = code.message_len
    threads = oracle.cpu_count()
    dec = HybridDecoder(code, BpConfig(i_max=IMAX), SclConfig(L), capacity=CHUNK)
    res = {}
    for i, eb in enumerate(EBNO):
        errs, scl = [], []
        for first in range(0, FRAMES, CHUNK):
            nb = min(CHUNK, FRAMES - first)
            msgs, llr32 = host_frames(POINT0 + i, eb, nb, threads, first)
            dec.run(torch.from_numpy(llr32).cuda(), nb).sync()
            r = dec.host_results()
            errs.append((nat.unpack_bits(r["payload"], m) != msgs).sum(axis=1).astype(np.uint16))
            scl.append(~r["converged"][:nb])
        res[f"err_{i}"] = np.concatenate(errs)
        res[f"scl_{i}"] = np.concatenate(scl)
        print(eb, "dB device frame errors", int((res[f"err_{i}"] > 0).sum()), flush=True)
    np.savez_compressed(out, **res)


def oracle_phase(dev_file, out):
    import oracle
    from paper_1609_09358_b200 import CodeConfig

    code = CodeConfig(N, K, crc=16)
    m = code.message_len
    threads = oracle.cpu_count()
    dev = np.load(dev_file)
    rep = {"config": f"hybrid N={N} K={K} (m={m}) L={L} i_max={IMAX}; {FRAMES} paired host frames per point "
                     f"(PCG64 keyed (31415, {POINT0}+i, frame), fp32-rounded LLRs); device = B200 pipeline, "
                     f"oracle = fp64 C port on {threads} threads", "points": []}
    ok = True
    for i, eb in enumerate(EBNO):
        t0 = time.time()
        dev_err, dev_scl = dev[f"err_{i}"].astype(np.int64), dev[f"scl_{i}"]
        ref_err, ref_scl = [], []
        for first in range(0, FRAMES, CHUNK):
            nb = min(CHUNK, FRAMES - first)
            msgs, llr32 = host_frames(POINT0 + i, eb, nb, threads, first)
            pay, prov, _ = oracle.hybrid_batch(llr32.astype(np.float64), code, i_max=IMAX, L=L, nthreads=threads)
            ref_err.append((pay != msgs).sum(axis=1))
            ref_scl.append(prov)
        ref_err, ref_scl = np.concatenate(ref_err), np.concatenate(ref_scl)
        fd, fr = int((dev_err > 0).sum()), int((ref_err > 0).sum())
        a = int(((dev_err > 0) & (ref_err == 0)).sum())
        b = int(((ref_err > 0) & (dev_err == 0)).sum())
        pval = 1.0 if a + b == 0 else min(1.0, sum(math.comb(a + b, j) for j in range(min(a, b) + 1)) / 2 ** (a + b - 1))
        lo, hi = clopper_pearson(fr, FRAMES)
        inside = lo <= fd / FRAMES <= hi
        ok &= inside and pval > 0.01
        pt = {"ebno_db": eb, "frames": FRAMES, "frame_errors_device": fd, "frame_errors_oracle": fr,
              "fer_device": fd / FRAMES, "fer_device_ci95": list(clopper_pearson(fd, FRAMES)),
              "fer_oracle": fr / FRAMES, "fer_oracle_ci95": [lo, hi], "device_fer_inside_oracle_ci": inside,
              "discordant_device_only": a, "discordant_oracle_only": b, "sign_test_p": pval,
              "to_scl_device": int(dev_scl.sum()), "to_scl_oracle": int(ref_scl.sum()),
              "provenance_flips": int((dev_scl != ref_scl).sum()),
              "errors_on_bp_accepted_frames_device": int(((dev_err > 0) & ~dev_scl).sum()),
              "errors_on_bp_accepted_frames_oracle": int(((ref_err > 0) & ~ref_scl).sum()),
              "ber_device": cluster_ci(dev_err, m), "ber_oracle": cluster_ci(ref_err, m),
              "oracle_seconds": time.time() - t0}
        rep["points"].append(pt)
        print(json.dumps(pt), flush=True)
    rep["all_points_pass"] = ok
    rep["note"] = ("errors_on_bp_accepted_frames = frame errors the CRC-16 stop accepted in BP (the false-accept "
                   "floor, probability ~2^-16 per check of a wrong estimate)")
    Path(out).write_text(json.dumps(rep, indent=1))
    print("ALL_OK" if ok else "MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("phase", choices=("device", "oracle"))
    ap.add_argument("files", nargs="+")
    ap.add_argument("--ebno", default=",".join(str(e) for e in EBNO))
    ap.add_argument("--frames", type=int, default=FRAMES)
    ap.add_argument("--point0", type=int, default=POINT0)
    args = ap.parse_args()
    EBNO = tuple(float(x) for x in args.ebno.split(","))
    FRAMES, POINT0 = args.frames, args.point0
    if args.phase == "device":
        device_phase(args.files[0])
    else:
        sys.exit(oracle_phase(args.files[0], args.files[1]))
