"""FER / BER parity of the device hybrid decoder against the fp64 CPU oracle.

For each Eb/N0 point, the same host frames (reference PCG64 keying,
fp32-rounded LLRs) are decoded by the device pipeline (K1 -> K2 -> K3) and by
the oracle port of the reference algorithm (all host threads).  Reported per
point:
  * FER of both on the paired frames, with exact Clopper-Pearson 95% CIs and
    the check "device FER inside the oracle's CI";
  * the paired discordance (frames only one side got wrong) with an exact
    two-sided sign-test p-value (reference test_acceptance.py:223-257);
  * BER with the reference's per-frame cluster CI (test_acceptance.py:55-61);
  * the device FER on a larger device-only sample (Philox frames), whose CI
    must overlap the oracle's.

    python tests/parity/fer_parity.py [--frames 2000] [--device-frames 131072] [--out profiles/fer_parity.json]

With --frames above --chunk (default 65536) the paired frames are generated,
decoded on both sides and counted chunk by chunk (10^6 paired frames per
point fit in host memory), e.g. the high-SNR floor check
    python tests/parity/fer_parity.py --frames 1000000 --ebno 3,3.5,4 --device-frames 0 \
        --out profiles/fer_parity_1e6.json
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

N, K, L, IMAX, SEED = 1024, 512, 32, 50, 31415


def clopper_pearson(k: int, n: int, alpha: float = 0.05):
    from scipy.stats import beta

    lo = 0.0 if k == 0 else float(beta.ppf(alpha / 2, k, n - k + 1))
    hi = 1.0 if k == n else float(beta.ppf(1 - alpha / 2, k + 1, n - k))
    return lo, hi


def cluster_ci(per_frame_errors, bits):
    e = np.asarray(per_frame_errors, dtype=np.float64)
    ber = e.sum() / (e.size * bits)
    se = e.std(ddof=1) / (math.sqrt(e.size) * bits) if e.size > 1 else 0.0
    return ber, ber - 1.96 * se, ber + 1.96 * se


def _frames(args):
    point, ebno, first, count = args
    from paper_1609_09358_b200 import CodeConfig
    from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame

    code = CodeConfig(N, K, crc=16)
    sigma = ebno_to_sigma(ebno, code.rate)
    out = [make_frame(code, sigma, frame_rng(SEED, point, f)) for f in range(first, first + count)]
    return np.array([o[0] for o in out]), np.array([o[1] for o in out]).astype(np.float32)


def _frames_batch(args):
    point, ebno, first, count = args
    from paper_1609_09358_b200 import CodeConfig
    from paper_1609_09358_b200.channel import ebno_to_sigma, make_frames

    code = CodeConfig(N, K, crc=16)
    msgs, llrs = make_frames(code, ebno_to_sigma(ebno, code.rate), SEED, point, first, count)
    return msgs, llrs.astype(np.float32)


def host_frames(point, ebno, count, workers, first=0):
    chunks = [(point, ebno, first + s, min(2048, count - s)) for s in range(0, count, 2048)]
    with ProcessPoolExecutor(workers) as ex:
        parts = list(ex.map(_frames_batch, chunks))
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=2000)
    ap.add_argument("--device-frames", type=int, default=131072)
    ap.add_argument("--ebno", default="1,1.5,2,2.5,3,3.5,4")
    ap.add_argument("--chunk", type=int, default=65536)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "fer_parity.json"))
    args = ap.parse_args()

    import torch

    import oracle
    from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig
    from paper_1609_09358_b200 import _native as nat
    from paper_1609_09358_b200.channel import ebno_to_sigma

    code = CodeConfig(N, K, crc=16)
    m = code.message_len
    threads = oracle.cpu_count()
    report = {"config": f"hybrid N={N} K={K} (m={m}) L={L} i_max={IMAX}; paired frames: host PCG64 keyed "
                        f"(seed {SEED}, point, frame), fp32-rounded LLRs; oracle = fp64 C port on {threads} threads",
              "points": []}
    all_ok = True
    for p, eb in enumerate(float(x) for x in args.ebno.split(",")):
        t0 = time.time()
        cap = max(min(args.frames, args.chunk), args.device_frames)
        dec = HybridDecoder(code, BpConfig(i_max=IMAX), SclConfig(L), capacity=cap)
        dev_err, ref_err, flips = [], [], 0
        t_oracle = 0.0
        for first in range(0, args.frames, args.chunk):
            nb = min(args.chunk, args.frames - first)
            msgs, llr32 = host_frames(p, eb, nb, threads, first)
            dec.run(torch.from_numpy(llr32).cuda(), nb).sync()
            r = dec.host_results()
            dev_pay = nat.unpack_bits(r["payload"], m)
            t1 = time.time()
            ref_pay, ref_prov, _ = oracle.hybrid_batch(llr32.astype(np.float64), code, i_max=IMAX, L=L,
                                                       nthreads=threads)
            t_oracle += time.time() - t1
            dev_err.append((dev_pay != msgs).sum(axis=1))
            ref_err.append((ref_pay != msgs).sum(axis=1))
            flips += int((~r["converged"][:nb] != ref_prov).sum())
        dev_err, ref_err = np.concatenate(dev_err), np.concatenate(ref_err)
        fd, fr = int((dev_err > 0).sum()), int((ref_err > 0).sum())
        lo, hi = clopper_pearson(fr, args.frames)
        a = int(((dev_err > 0) & (ref_err == 0)).sum())
        b = int(((ref_err > 0) & (dev_err == 0)).sum())
        pval = 1.0 if a + b == 0 else min(1.0, sum(math.comb(a + b, i) for i in range(min(a, b) + 1)) / 2 ** (a + b - 1))
        ber_d = cluster_ci(dev_err, m)
        ber_r = cluster_ci(ref_err, m)
        # larger device-only sample (Philox frames)
        B = args.device_frames
        if B == 0:
            inside = lo <= fd / args.frames <= hi
            all_ok &= inside and pval > 0.01
            pt = {"ebno_db": eb, "frames": args.frames, "frame_errors_device": fd, "frame_errors_oracle": fr,
                  "fer_device": fd / args.frames, "fer_oracle": fr / args.frames, "fer_oracle_ci95": [lo, hi],
                  "fer_device_ci95": list(clopper_pearson(fd, args.frames)), "device_fer_inside_oracle_ci": inside,
                  "discordant_device_only": a, "discordant_oracle_only": b, "sign_test_p": pval,
                  "provenance_flips": flips, "ber_device": ber_d, "ber_oracle": ber_r,
                  "oracle_seconds": t_oracle, "seconds": time.time() - t0}
            report["points"].append(pt)
            print(json.dumps(pt), flush=True)
            continue
        llr = torch.empty((B, N), dtype=torch.float32, device="cuda")
        mw = torch.empty((B, (m + 31) // 32), dtype=torch.int32, device="cuda")
        dc = nat.device_code(code)
        lib = nat.load()
        nat.check(lib.pc_gen_frames(SEED, p, 0, B, ebno_to_sigma(eb, code.rate), dc.ref, mw.data_ptr(), llr.data_ptr(),
                                    nat.stream_handle()), "gen")
        dec.run(llr, B).sync()
        cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
        nat.check(lib.pc_count_errors(dec.payload.data_ptr(), mw.data_ptr(), B, m, cnt.data_ptr(), nat.stream_handle()),
                  "count")
        big_fe = int(cnt[1].item())
        blo, bhi = clopper_pearson(big_fe, B)
        inside = lo <= fd / args.frames <= hi
        overlap = not (bhi < lo or blo > hi)
        all_ok &= inside and overlap and pval > 0.01
        pt = {
            "ebno_db": eb, "frames": args.frames,
            "fer_device": fd / args.frames, "fer_oracle": fr / args.frames, "fer_oracle_ci95": [lo, hi],
            "device_fer_inside_oracle_ci": inside,
            "discordant_device_only": a, "discordant_oracle_only": b, "sign_test_p": pval,
            "provenance_flips": flips,
            "ber_device": ber_d, "ber_oracle": ber_r,
            "device_only": {"frames": B, "fer": big_fe / B, "fer_ci95": [blo, bhi], "overlaps_oracle_ci": overlap},
            "seconds": time.time() - t0,
        }
        report["points"].append(pt)
        print(json.dumps(pt), flush=True)
    report["all_points_pass"] = all_ok
    Path(args.out).write_text(json.dumps(report, indent=1))
    print("ALL_OK" if all_ok else "MISMATCH", flush=True)
    return 0 if all_ok else 1


if __name__ == "__main__":
    sys.exit(main())
