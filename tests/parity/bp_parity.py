"""C1 / C4 BP decisions at scale against the fp64 oracle (BASELINE configs[0]
N=128 K=64 at 2 dB; configs[3] N=4096 K=2048 at 2 and 3 dB), CRC stop,
i_max=50, on the same host frames (reference PCG64 keying, fp32-rounded
LLRs).  Per set: frames whose (converged, iterations, u_hat) agree; the
differing ones split into "early" (the reference decides within 20
iterations: must be certified near-ties, tests/test_gpu_bp.py) and "late"
(the fp32/fp64 divergence class).  The early ones are certified here with the
same two criteria as the test suite.

    python tests/parity/bp_parity.py [--frames 10000] [--out profiles/bp_parity.json]
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
sys.path.insert(0, str(ROOT / "tests"))

SEED = 16180


def frames(code, eb, count, point, workers):
    from concurrent.futures import ProcessPoolExecutor

    chunks = [(code.N, code.k, eb, point, s, min(256, count - s)) for s in range(0, count, 256)]
    with ProcessPoolExecutor(workers) as ex:
        parts = list(ex.map(_chunk, chunks))
    return np.concatenate(parts).astype(np.float32).astype(np.float64)


def _chunk(args):
    N, k, eb, point, first, count = args
    from paper_1609_09358_b200 import CodeConfig
    from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame

    code = CodeConfig(N, k, crc=16)
    sigma = ebno_to_sigma(eb, code.rate)
    return np.array([make_frame(code, sigma, frame_rng(SEED, point, f))[1] for f in range(first, first + count)])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=10000)
    ap.add_argument("--frames4096", type=int, default=2000)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "bp_parity.json"))
    args = ap.parse_args()

    import oracle
    from test_gpu_bp import ill_conditioned, near_tie

    from paper_1609_09358_b200 import BpConfig, CodeConfig, bp_decode_batch

    threads = oracle.cpu_count()
    report = {"config": f"BP i_max=50 exact g, CRC-16 stop; host PCG64 frames (seed {SEED}), fp32-rounded LLRs; "
                        f"oracle = fp64 C port on {threads} threads", "sets": []}
    ok_all = True
    for name, N, k, eb, count, point in (("C1", 128, 64, 2.0, args.frames, 0),
                                         ("C4-2dB", 4096, 2048, 2.0, args.frames4096, 1),
                                         ("C4-3dB", 4096, 2048, 3.0, args.frames4096, 2)):
        t0 = time.time()
        code = CodeConfig(N, k, crc=16)
        llrs = frames(code, eb, count, point, threads)
        ref_u, ref_it, ref_cv = oracle.bp_batch(llrs, code, stop_mode="crc", nthreads=threads)
        got = bp_decode_batch(llrs, code, BpConfig(stop_mode="crc"))
        same = (got.converged == ref_cv) & (got.iterations_used == ref_it)
        same &= np.array([not ref_cv[f] or np.array_equal(got.u_hat[f], ref_u[f]) for f in range(count)])
        diff = np.flatnonzero(~same)
        early = [int(f) for f in diff if ref_it[f] <= 20]
        late = [int(f) for f in diff if ref_it[f] > 20]
        certified, uncertified = [], []
        for f in early:
            kk = min(int(ref_it[f]), int(got.iterations_used[f]))
            dev_k = bp_decode_batch(llrs[f:f + 1], code, BpConfig(i_max=kk, stop_mode="none"))
            okc, _ = near_tie(llrs[f], code, kk, dev_k.u_hat[0])
            (certified if okc or ill_conditioned(llrs[f], code, int(ref_it[f]), ref_cv[f]) else uncertified).append(f)
        ok_all &= not uncertified
        row = {"set": name, "N": N, "ebno_db": eb, "frames": count, "identical": int(same.sum()),
               "differing_early_certified": len(certified), "differing_early_uncertified": uncertified,
               "differing_late": len(late), "mean_iterations_ref": float(ref_it.mean()),
               "mean_iterations_dev": float(np.asarray(got.iterations_used).mean()),
               "fer_bp_ref": float(1 - ref_cv.mean()), "fer_bp_dev": float(1 - np.asarray(got.converged).mean()),
               "seconds": time.time() - t0}
        report["sets"].append(row)
        print(json.dumps(row), flush=True)
    report["all_certified"] = ok_all
    Path(args.out).write_text(json.dumps(report, indent=1))
    print("ALL_OK" if ok_all else "UNCERTIFIED")
    return 0 if ok_all else 1


if __name__ == "__main__":
    sys.exit(main())
