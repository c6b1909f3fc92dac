"""Precision study for K1 in the likelihood-ratio domain.

Messages as Lambda = e^v (fp32) instead of LLRs v: a sum of LLRs is a product,
the exact node update is g = (1 + Lx Ly) / (Lx + Ly) (bp.py:86-100), so a PE
needs two reciprocals and no exp/log.  The clip |v| <= 20 bounds Lambda to
[e^-20, e^20] (sums to e^40), well inside fp32.  This emulates that arithmetic
in numpy fp32 (exactly rounded reciprocal; the device's rcp.approx is within
1 ulp) over a batch of frames and compares (converged, iterations, u_hat) with
the fp64 oracle, the same split as tests/parity/bp_parity.py.

    python tools/lr_domain_study.py N K ebno frames
"""

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "parity"))

f32 = np.float32


def bp_lr_f32(llrs, code, i_max=50, llr_max=20.0, recip=None, stop=True):
    F, N, n = llrs.shape[0], code.N, code.n
    hi, lo = f32(np.exp(llr_max)), f32(np.exp(-llr_max))
    L = np.ones((n + 1, F, N), f32)
    R = np.ones((n + 1, F, N), f32)
    L[n] = np.exp(np.clip(llrs.astype(f32), -llr_max, llr_max).astype(np.float64)).astype(f32)
    R[0] = np.where(np.asarray(code.frozen_mask, bool), hi, f32(1))[None, :]
    rc = recip or (lambda x: (f32(1) / x).astype(f32))

    def g(x, y):
        return (np.float32(1) + x * y) * rc(x + y)

    info = np.asarray(code.info_positions)
    crc_cols = None
    from paper_1609_09358_b200.codes import crc_check

    it_used = np.full(F, i_max, np.int32)
    conv = np.zeros(F, bool)
    u_fin = np.zeros((F, N), np.uint8)
    active = np.arange(F)
    for it in range(1, i_max + 1):
        for j in range(1, n + 1):
            h = 1 << (j - 1)
            Rp, Lj = R[j - 1].reshape(F, -1, 2, h), L[j].reshape(F, -1, 2, h)
            a, r2, l1, l2 = Rp[:, :, 0], Rp[:, :, 1], Lj[:, :, 0], Lj[:, :, 1]
            o = R[j].reshape(F, -1, 2, h)
            o1 = g(a, l2 * r2)
            o2 = np.clip(g(a, l1) * r2, lo, hi)
            o[:, :, 0], o[:, :, 1] = o1, o2
        for j in range(n, 0, -1):
            h = 1 << (j - 1)
            Rp, Lj = R[j - 1].reshape(F, -1, 2, h), L[j].reshape(F, -1, 2, h)
            a, r2, l1, l2 = Rp[:, :, 0], Rp[:, :, 1], Lj[:, :, 0], Lj[:, :, 1]
            o = L[j - 1].reshape(F, -1, 2, h)
            o1 = g(l1, l2 * r2)
            o2 = np.clip(g(a, l1) * l2, lo, hi)
            o[:, :, 0], o[:, :, 1] = o1, o2
        su = L[0] * R[0]
        u = (su < 1).astype(np.uint8)
        for f in (np.flatnonzero(~conv) if stop else []):
            if crc_check(u[f][info], code.crc):
                conv[f] = True
                it_used[f] = it
                u_fin[f] = u[f]
        if conv.all():
            break
    for f in np.flatnonzero(~conv):
        u_fin[f] = u[f]
    return u_fin, it_used, conv


def main():
    N, K, eb, count = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
    import oracle
    from bp_parity import frames

    from paper_1609_09358_b200 import CodeConfig

    code = CodeConfig(N, K, crc=16)
    threads = oracle.cpu_count()
    llrs = frames(code, eb, count, 7, threads)
    t0 = time.time()
    ref_u, ref_it, ref_cv = oracle.bp_batch(llrs, code, stop_mode="crc", nthreads=threads)
    t1 = time.time()
    u, it, cv = bp_lr_f32(llrs, code)
    t2 = time.time()
    same = (cv == ref_cv) & (it == ref_it)
    same &= np.array([not ref_cv[f] or np.array_equal(u[f], ref_u[f]) for f in range(count)])
    diff = np.flatnonzero(~same)
    early = [int(f) for f in diff if ref_it[f] <= 20]
    sys.path.insert(0, str(ROOT / "tests"))
    from test_gpu_bp import ill_conditioned, near_tie

    cert = []
    for f in early:
        kk = min(int(ref_it[f]), int(it[f]))
        uk, _, _ = bp_lr_f32(llrs[f:f + 1], code, i_max=kk, stop=False)
        ok, worst = near_tie(llrs[f], code, kk, uk[0])
        cert.append((f, ok or ill_conditioned(llrs[f], code, int(ref_it[f]), ref_cv[f]), worst))
    print("early certification:", cert)
    print(f"N={N} K={K} {eb} dB frames={count}: identical {same.sum()}, early {len(early)} {early[:10]}, "
          f"late {len(diff) - len(early)}; mean it ref {ref_it.mean():.3f} lr {it.mean():.3f}; "
          f"FER_bp ref {1 - ref_cv.mean():.4f} lr {1 - cv.mean():.4f}  ({t1 - t0:.1f}s oracle, {t2 - t1:.1f}s lr)")


if __name__ == "__main__":
    main()
