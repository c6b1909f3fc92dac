"""Test utility: a literal float32 restatement of the reference BP with the
min-sum node update (bp.py:86-100, 138-161, 176-208), numpy, per frame.

Min-sum BP has no smoothing, so fp32 and fp64 runs drift apart after ~10-20
iterations at N=4096 (rounding of the sums l2 + r2 and g + r2 is amplified;
SURVEY.md section 7 hard part 2).  The device's min-sum arithmetic is exactly
this fp32 sequence (min, sign, clip and one fp32 rounding per add), so the
device must agree with it BIT-EXACTLY; the fp64 oracle is the reference for
the exact-g mode.  Test-only: never imported by the package.
"""

import numpy as np

from paper_1609_09358_b200.codes import crc_check


def _g_min(a, b, lim):
    m = np.minimum(np.abs(a), np.abs(b))
    mag = np.where((a == 0) | (b == 0), np.float32(0), m)
    return np.clip(np.sign(a) * np.sign(b) * mag, -lim, lim).astype(np.float32)


def bp_minsum_f32(llr, code, i_max=50, llr_max=20.0):
    """(u_hat, iterations_used, converged) with the CRC stop after every iteration."""
    N, n = code.N, code.n
    lim = np.float32(llr_max)
    L = np.zeros((n + 1, N), np.float32)
    R = np.zeros((n + 1, N), np.float32)
    L[n] = np.clip(np.asarray(llr, np.float32), -lim, lim)
    R[0] = lim * np.asarray(code.frozen_mask, np.float32)
    info = np.asarray(code.info_positions)
    u = np.zeros(N, np.uint8)
    for it in range(1, i_max + 1):
        for j in range(1, n + 1):
            h = 1 << (j - 1)
            Rp, Lj, Rd = R[j - 1].reshape(-1, 2, h), L[j].reshape(-1, 2, h), R[j].reshape(-1, 2, h)
            a, r2, l1, l2 = Rp[:, 0].copy(), Rp[:, 1].copy(), Lj[:, 0].copy(), Lj[:, 1].copy()
            Rd[:, 0] = _g_min(a, l2 + r2, lim)
            Rd[:, 1] = np.clip(_g_min(a, l1, lim) + r2, -lim, lim)
        for j in range(n, 0, -1):
            h = 1 << (j - 1)
            Rp, Lj, Ld = R[j - 1].reshape(-1, 2, h), L[j].reshape(-1, 2, h), L[j - 1].reshape(-1, 2, h)
            a, r2, l1, l2 = Rp[:, 0].copy(), Rp[:, 1].copy(), Lj[:, 0].copy(), Lj[:, 1].copy()
            Ld[:, 0] = _g_min(l1, l2 + r2, lim)
            Ld[:, 1] = np.clip(_g_min(a, l1, lim) + l2, -lim, lim)
        u = ((L[0] + R[0]) < 0).astype(np.uint8)
        if crc_check(u[info], code.crc):
            return u, it, True
    return u, i_max, False
