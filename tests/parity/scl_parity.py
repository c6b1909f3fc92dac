"""C2 / C5 at scale (BASELINE configs[1]: CRC-aided SCL L=32, N=1024 K=512,
"bit-exact vs the CPU reference on shared LLR inputs"; configs[4]: N=2048
K=1024, L = 1..32 at 2 dB): the device list decoder against the fp64 oracle
on the same host frames (reference PCG64 keying, fp32-rounded LLRs), per row:
winners (u_hat), CRC flags and metrics (relative difference).

    python tests/parity/scl_parity.py [--frames 10000] [--out profiles/scl_parity_c2.json]
    python tests/parity/scl_parity.py --c5 [--frames 10000] [--out profiles/scl_parity_c5.json]
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

import fer_parity  # noqa: E402  (host frame generation, same keying)

N, K, L, SEED = 1024, 512, 32, 27182


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=10000)
    ap.add_argument("--ebno", default="1,1.5,2,2.5,3,3.5,4")
    ap.add_argument("--out", default=None)
    ap.add_argument("--c5", action="store_true", help="N=2048 K=1024 at 2 dB, L = 1..32")
    args = ap.parse_args()
    global N, K
    if args.c5:
        N, K = 2048, 1024
        fer_parity.N, fer_parity.K = N, K
        rows = [(L_, 2.0) for L_ in (1, 2, 4, 8, 16, 32)]
    else:
        rows = [(L, float(x)) for x in args.ebno.split(",")]
    out = args.out or str(ROOT / "profiles" / ("scl_parity_c5.json" if args.c5 else "scl_parity_c2.json"))

    import oracle
    from paper_1609_09358_b200 import CodeConfig, SclConfig, scl_decode_batch

    fer_parity.SEED = SEED
    code = CodeConfig(N, K, crc=16)
    threads = oracle.cpu_count()
    report = {"config": f"CRC-aided SCL N={N} K={K} (exact metric, min-sum f, pseudo selector); host PCG64 "
                        f"frames (seed {SEED}), fp32-rounded LLRs; oracle = fp64 C port on {threads} threads",
              "points": []}
    total_bad = 0
    for p, (Lr, eb) in enumerate(rows):
        t0 = time.time()
        msgs, llr32 = fer_parity.host_frames(0 if args.c5 else p, eb, args.frames, threads)
        llr = llr32.astype(np.float64)
        got = scl_decode_batch(llr, code, SclConfig(Lr))
        ref_u, ref_m, ref_ok = oracle.scl_batch(llr, code, Lr, nthreads=threads)
        same_u = (got.u_hat == ref_u).all(axis=1)
        same_ok = got.crc_ok == ref_ok
        rel = np.abs(got.metric - ref_m) / np.maximum(np.abs(ref_m), 1.0)
        bad = int((~(same_u & same_ok)).sum())
        total_bad += bad
        pay = got.u_hat[:, np.asarray(code.info_positions)[:code.message_len]]
        fer = float((pay != msgs).any(axis=1).mean())
        row = {"L": Lr, "ebno_db": eb, "frames": args.frames, "winners_differing": bad, "crc_flags_differing": int((~same_ok).sum()),
               "metric_max_rel_diff": float(rel.max()), "fer": fer, "seconds": time.time() - t0}
        report["points"].append(row)
        print(json.dumps(row), flush=True)
    report["winners_differing_total"] = total_bad
    Path(out).write_text(json.dumps(report, indent=1))
    print("ALL_IDENTICAL" if total_bad == 0 else f"DIFFERING {total_bad}")
    return 0 if total_bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
