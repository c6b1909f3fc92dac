"""Certify the SCL winners that differ at 10^6 frames per point (C2, N=1024
K=512 L=32; tests/parity/scl_parity.py --frames 1000000): same frames (PCG64
keying of scl_parity.py, fp32-rounded LLRs), decoded in chunks on the device
and by the oracle; for every differing frame the reference's closest list
selection (oracle.scl_min_margin) is compared with the fp32 rounding of a
metric summed over that many leaves (fuzz_parity.selection_limited).

    python tests/parity/scl_certify.py gpurun_out/scl_certify.json [--ebno 1,1.5,2] [--frames 1000000]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import fer_parity  # noqa: E402

N, K, L, SEED, CHUNK = 1024, 512, 32, 27182, 65536
POINT_OF = {1.0: 0, 1.5: 1, 2.0: 2, 2.5: 3, 3.0: 4, 3.5: 5, 4.0: 6}  # scl_parity.py's point keys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--ebno", default="1,1.5,2")
    ap.add_argument("--frames", type=int, default=1000000)
    a = ap.parse_args()
    import oracle
    from paper_1609_09358_b200 import CodeConfig, SclConfig, scl_decode_batch

    fer_parity.SEED = SEED
    code = CodeConfig(N, K, crc=16)
    threads = oracle.cpu_count()
    rep = {"config": f"C2 N={N} K={K} L={L}, frames of tests/parity/scl_parity.py (seed {SEED}), {a.frames} per point",
           "points": []}
    for eb in (float(x) for x in a.ebno.split(",")):
        t0 = time.time()
        p = POINT_OF[eb]
        diff = []
        for first in range(0, a.frames, CHUNK):
            nb = min(CHUNK, a.frames - first)
            _, llr32 = fer_parity.host_frames(p, eb, nb, threads, first)
            llr = llr32.astype(np.float64)
            got = scl_decode_batch(llr, code, SclConfig(L))
            ref_u, _, ref_ok = oracle.scl_batch(llr, code, L, nthreads=threads)
            bad = np.flatnonzero(~((got.u_hat == ref_u).all(axis=1) & (got.crc_ok == ref_ok)))
            for f in bad:
                gap, metric, leaf = oracle.scl_min_margin(llr[f], code, L)
                tol = 0.5 * (leaf + 1) * float(np.spacing(np.float32(abs(metric))))
                diff.append({"frame": int(first + f), "gap": float(gap), "metric": float(metric), "leaf": int(leaf),
                             "fp32_tolerance": tol, "selection_limited": bool(leaf >= 0 and gap < tol)})
        pt = {"ebno_db": eb, "frames": a.frames, "differing": len(diff),
              "certified_selection_limited": sum(d["selection_limited"] for d in diff), "frames_differing": diff,
              "seconds": time.time() - t0}
        rep["points"].append(pt)
        print(json.dumps({k: v for k, v in pt.items() if k != "frames_differing"}), flush=True)
    Path(a.out).write_text(json.dumps(rep, indent=1))
    ok = all(p["differing"] == p["certified_selection_limited"] for p in rep["points"])
    print("ALL_CERTIFIED" if ok else "UNCERTIFIED")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
