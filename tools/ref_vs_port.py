"""The untouched Python reference (polarsim, imported from /root/reference in
THIS container only) beside the oracle port (oracle/oracle.c), on the same
host frames and the same host cores: P processes of
the reference, each decoding a disjoint frame range of every Eb/N0 point with
hybrid_decode_batch(BpConfig(i_max=50), SclConfig(32), bp_batch_size=32,
n_scl_workers=1), decode-only wall; then the port on P threads over the same
frames.  Output: profiles/ref_vs_port.json (both throughputs, their ratio,
and whether the decoded payloads agree).

    python tools/ref_vs_port.py [frames_per_point] [processes]
"""
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
EBNO = (1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0)
SEED = 20240917


def _ref_worker(args):
    """One reference process: frames [lo, hi) of every point, reference API only."""
    lo, hi = args
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(REF))
    import polarsim as ps
    from polarsim.sim import _make_frame

    code = ps.CodeConfig(1024, 512, crc=16)
    # warm the JIT and the CRC tables on a throwaway frame
    m, l = _make_frame(code, ps.ebno_to_sigma(2.0, code.rate), ps.frame_rng(1, 99, 0))
    ps.hybrid_decode_batch([ps.FrameJob(frame_id=0, llrs=l, true_message=m)], code, ps.BpConfig(i_max=50),
                           ps.SclConfig(32), bp_batch_size=32, n_scl_workers=1)
    ps.scl_decode(l, code, ps.SclConfig(32))  # the numba SCL kernel's JIT (the frame above may stop in BP)
    out = []
    for p, eb in enumerate(EBNO):
        sigma = ps.ebno_to_sigma(eb, code.rate)
        jobs = []
        for f in range(lo, hi):
            m, l = _make_frame(code, sigma, ps.frame_rng(SEED, p, f))
            jobs.append(ps.FrameJob(frame_id=f, llrs=l, true_message=m))
        t = time.perf_counter()
        ps.hybrid_decode_batch(jobs, code, ps.BpConfig(i_max=50), ps.SclConfig(32), bp_batch_size=32,
                               n_scl_workers=1)
        dt = time.perf_counter() - t
        out.append((dt, np.array([j.message for j in jobs]), np.array([j.provenance == "scl" for j in jobs])))
    return out


def main():
    fpp = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    P = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
    sys.path.insert(0, str(ROOT))
    import oracle
    from paper_1609_09358_b200 import CodeConfig
    from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame

    code = CodeConfig(1024, 512, crc=16)
    m = code.message_len
    bounds = [(fpp * r // P, fpp * (r + 1) // P) for r in range(P)]
    with ProcessPoolExecutor(P) as ex:
        parts = list(ex.map(_ref_worker, bounds))
    rows = []
    ref_wall_total, port_wall_total = 0.0, 0.0
    for p, eb in enumerate(EBNO):
        ref_wall = max(part[p][0] for part in parts)  # max per-process decode wall
        ref_pay = np.concatenate([part[p][1] for part in parts])
        ref_prov = np.concatenate([part[p][2] for part in parts])
        sigma = ebno_to_sigma(eb, code.rate)
        llrs = np.array([make_frame(code, sigma, frame_rng(SEED, p, f))[1] for f in range(fpp)])
        t = time.perf_counter()
        pay, prov, _ = oracle.hybrid_batch(llrs, code, i_max=50, L=32, nthreads=P)
        port_wall = time.perf_counter() - t
        ref_wall_total += ref_wall
        port_wall_total += port_wall
        rows.append({"ebno_db": eb, "frames": fpp, "reference_s": ref_wall, "port_s": port_wall,
                     "reference_mbps": fpp * m / ref_wall / 1e6, "port_mbps": fpp * m / port_wall / 1e6,
                     "payload_frames_identical": int((pay == ref_pay).all(axis=1).sum()),
                     "provenance_identical": int((prov == ref_prov).sum())})
        print(json.dumps(rows[-1]), flush=True)
    ref_v = len(EBNO) * fpp * m / ref_wall_total / 1e9
    port_v = len(EBNO) * fpp * m / port_wall_total / 1e9
    rep = {"what": "untouched Python reference (polarsim, P processes, hybrid_decode_batch bp_batch_size=32 "
                   "n_scl_workers=1, decode-only wall = max over processes) vs the fp64 C port (oracle.hybrid_batch, "
                   "P threads) on the same host frames, N=1024 K=512 CRC-16 L=32 i_max=50, Eb/N0 1-4 dB",
           "host": f"{os.cpu_count()} logical CPUs (dev container, not the B200 box)", "processes": P,
           "frames_per_point": fpp, "reference_gbps": ref_v, "port_gbps": port_v, "port_over_reference": port_v / ref_v,
           "points": rows}
    (ROOT / "profiles" / "ref_vs_port.json").write_text(json.dumps(rep, indent=1))
    print(json.dumps({k: rep[k] for k in ("reference_gbps", "port_gbps", "port_over_reference")}))


if __name__ == "__main__":
    main()
