"""Generate tests/golden/*.npz|json from the REFERENCE package (run in the dev container).

    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything here comes from the unmodified reference `polarsim`
(/root/reference/pkg/src/polarsim) imported read-only.  The fixtures pin the
CPU oracle (oracle/oracle.c) and the host code-construction module, and are
the expected outputs the GPU parity tests compare against.  Frames are stored
as PCG64 keys (seed, point, frame, Eb/N0) plus a few literal LLR vectors that
pin the host frame generator; the LLRs fed to the decoders are the float32
roundings of the reference's float64 LLRs (the GPU computes in fp32), and the
reference decodes exactly those rounded values.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import polarsim as ref  # noqa: E402

OUT = Path(__file__).resolve().parent


def packbits(bits):
    return np.packbits(np.asarray(bits, np.uint8), axis=-1, bitorder="little")


def frames(code, ebno, seed, point, count, first=0):
    sigma = ref.ebno_to_sigma(ebno, code.rate)
    msgs, llrs = [], []
    for f in range(first, first + count):
        m, l = ref.sim._make_frame(code, sigma, ref.frame_rng(seed, point, f))
        msgs.append(m)
        llrs.append(l.astype(np.float32).astype(np.float64))
    return np.array(msgs), np.array(llrs)


def main():
    g = {}
    # ---- code construction -------------------------------------------------
    cons = [(8, 4, None), (16, 8, None), (64, 32, 8), (128, 64, 16), (256, 128, 16), (1024, 512, 16),
            (2048, 1024, 16), (4096, 2048, 16), (1024, 700, 24)]
    for N, k, crc in cons:
        c = ref.CodeConfig(N, k, crc=crc)
        g[f"mask_{N}_{k}"] = packbits(c.frozen_mask)
    # ---- CRC known answers ---------------------------------------------------
    rng = np.random.default_rng(7)
    crc_cases = []
    for w in (8, 16, 24):
        spec = ref.CrcSpec.standard(w)
        for L in (1, 17, 48, 496, 1008):
            m = rng.integers(0, 2, L).astype(np.uint8)
            crc_cases.append((w, m, ref.crc_compute(m, spec)))
    g["crc_widths"] = np.array([c[0] for c in crc_cases])
    g["crc_msgs"] = np.array([packbits(np.pad(c[1], (0, 1008 - c[1].size))) for c in crc_cases])
    g["crc_lens"] = np.array([c[1].size for c in crc_cases])
    g["crc_out"] = np.array([packbits(np.pad(c[2], (0, 24 - c[2].size))) for c in crc_cases])
    # ---- encoder: insert_message + transform at N = 1024 ----------------------
    code = ref.CodeConfig(1024, 512, crc=16)
    msgs = rng.integers(0, 2, (16, code.message_len)).astype(np.uint8)
    g["enc_msgs"] = packbits(msgs)
    g["enc_x"] = packbits(np.array([ref.polar_transform(ref.insert_message(m, code)) for m in msgs]))
    # ---- host frame generator pin (literal fp64 LLRs) -------------------------
    m2, l2 = [], []
    for f in range(3):
        mm, ll = ref.sim._make_frame(code, ref.ebno_to_sigma(2.0, code.rate), ref.frame_rng(99, 1, f))
        m2.append(mm)
        l2.append(ll)
    g["gen_msgs"] = packbits(np.array(m2))
    g["gen_llrs"] = np.array(l2)

    # ---- BP with the CRC stop -------------------------------------------------
    bp_sets = [("bp128", 128, 64, 2.0, 11, 300), ("bp1024a", 1024, 512, 1.5, 12, 60),
               ("bp1024b", 1024, 512, 2.5, 13, 60), ("bp2048", 2048, 1024, 2.0, 14, 12),
               ("bp4096", 4096, 2048, 2.0, 17, 16)]
    meta = {}
    for name, N, k, eb, seed, cnt in bp_sets:
        c = ref.CodeConfig(N, k, crc=16)
        _, L = frames(c, eb, seed, 0, cnt)
        us, its, cv = [], [], []
        for l in L:
            r = ref.bp_decode(l, c, ref.BpConfig(i_max=50, stop_mode="crc"))
            us.append(r.u_hat)
            its.append(r.iterations_used)
            cv.append(r.converged)
        g[f"{name}_u"] = packbits(np.array(us))
        g[f"{name}_iters"] = np.array(its)
        g[f"{name}_conv"] = np.array(cv)
        meta[name] = dict(N=N, k=k, ebno=eb, seed=seed, point=0, count=cnt)
    # one re-encode / none stop-mode set on a small code without CRC
    c = ref.CodeConfig(64, 32, crc=None)
    _, L = frames(c, 2.0, 15, 0, 40)
    for mode in ("reencode", "none"):
        res = [ref.bp_decode(l, c, ref.BpConfig(i_max=20, stop_mode=mode)) for l in L]
        g[f"bp64_{mode}_u"] = packbits(np.array([r.u_hat for r in res]))
        g[f"bp64_{mode}_iters"] = np.array([r.iterations_used for r in res])
        g[f"bp64_{mode}_conv"] = np.array([r.converged for r in res])
    meta["bp64"] = dict(N=64, k=32, ebno=2.0, seed=15, point=0, count=40)

    # ---- BP teacher-forced iteration (fp64 reference, exact inputs) -----------
    for N, k, its in ((32, 16, 3), (1024, 512, 5)):
        c = ref.CodeConfig(N, k, crc=None)
        _, L = frames(c, 1.5, 16, 0, 1)
        cfg = ref.BpConfig(stop_mode="none")
        gr = ref.init_graph(L[0], c, cfg)
        for _ in range(its):
            ref.iterate_once(gr, c, cfg)
        lin = gr.l_msgs.astype(np.float32).astype(np.float64)
        rin = gr.r_msgs.astype(np.float32).astype(np.float64)
        gr2 = ref.BpGraph(lin.copy(), rin.copy())
        ref.iterate_once(gr2, c, cfg)
        g[f"tf{N}_lin"], g[f"tf{N}_rin"] = lin, rin
        g[f"tf{N}_lout"], g[f"tf{N}_rout"] = gr2.l_msgs, gr2.r_msgs

    # ---- SCL ------------------------------------------------------------------
    scl_sets = [("scl128L4", 128, 64, 4, 1.5, 21, 200), ("scl128L32", 128, 64, 32, 1.0, 22, 100),
                ("scl1024L8", 1024, 512, 8, 1.5, 23, 40), ("scl1024L32", 1024, 512, 32, 1.5, 24, 40),
                ("scl2048L32", 2048, 1024, 32, 2.0, 25, 8), ("scl256L1", 256, 128, 1, 1.0, 26, 100),
                ("scl512L2", 512, 256, 2, 1.5, 27, 60), ("scl512L16", 512, 256, 16, 1.5, 28, 30),
                ("scl2048L1", 2048, 1024, 1, 1.5, 33, 30), ("scl2048L4", 2048, 1024, 4, 1.5, 34, 20),
                ("scl4096L8", 4096, 2048, 8, 1.5, 35, 6)]
    for name, N, k, Lsz, eb, seed, cnt in scl_sets:
        c = ref.CodeConfig(N, k, crc=16)
        _, L = frames(c, eb, seed, 0, cnt)
        res = [ref.scl_decode(l, c, ref.SclConfig(list_size=Lsz)) for l in L]
        g[f"{name}_u"] = packbits(np.array([r.u_hat for r in res]))
        g[f"{name}_metric"] = np.array([r.metric for r in res])
        g[f"{name}_crc"] = np.array([r.crc_ok for r in res])
        meta[name] = dict(N=N, k=k, L=Lsz, ebno=eb, seed=seed, point=0, count=cnt)
    # knobs: exact f, approx metric, DA, CRC-8 at N=128
    c = ref.CodeConfig(128, 64, crc=8)
    _, L = frames(c, 1.5, 29, 0, 40)
    for tag, cfg in (("fexact", ref.SclConfig(8, f_mode="exact")), ("approx", ref.SclConfig(8, metric_mode="approx")),
                     ("da", ref.SclConfig(8, da_threshold=0.05))):
        res = [ref.scl_decode(l, c, cfg) for l in L]
        g[f"sclknob_{tag}_u"] = packbits(np.array([r.u_hat for r in res]))
        g[f"sclknob_{tag}_metric"] = np.array([r.metric for r in res])
    meta["sclknob"] = dict(N=128, k=64, crc=8, ebno=1.5, seed=29, point=0, count=40)

    # ---- hybrid ---------------------------------------------------------------
    for name, eb, seed, cnt in (("hyb1024a", 1.5, 31, 60), ("hyb1024b", 2.0, 32, 60)):
        c = ref.CodeConfig(1024, 512, crc=16)
        _, L = frames(c, eb, seed, 0, cnt)
        out = [ref.hybrid_decode_frame(l, c, ref.BpConfig(i_max=50), ref.SclConfig(32)) for l in L]
        g[f"{name}_payload"] = packbits(np.array([o[0] for o in out]))
        g[f"{name}_scl"] = np.array([o[1] == "scl" for o in out])
        meta[name] = dict(N=1024, k=512, L=32, ebno=eb, seed=seed, point=0, count=cnt)

    np.savez_compressed(OUT / "golden.npz", **g)
    # ---- the reference's committed simulator fixtures (non-timing columns) ----
    fx = {}
    fdir = Path("/root/reference/pkg/plot-tool/tests/fixtures")
    for p in sorted(fdir.glob("*.csv")):
        lines = p.read_text().splitlines()
        cfgline = [l for l in lines if l.startswith("# config: ")][0][len("# config: "):]
        rows = []
        hdr = None
        for l in lines:
            if l.startswith("#"):
                continue
            if hdr is None:
                hdr = l.split(",")
                continue
            cells = dict(zip(hdr, l.split(",")))
            rows.append({k: cells[k] for k in ("ebno_db", "frames", "bit_errors", "frame_errors", "gamma_bp_fer")})
        fx[p.stem] = dict(config=cfgline, rows=rows)
        if p.stem == "no_timing":  # byte-identity target for the CLI (--no-timing)
            fx[p.stem]["raw"] = p.read_text()
    (OUT / "golden_meta.json").write_text(json.dumps(dict(sets=meta, fixtures=fx), indent=1, sort_keys=True))
    print("wrote", OUT / "golden.npz", (OUT / "golden.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
