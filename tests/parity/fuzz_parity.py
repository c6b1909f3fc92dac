"""Randomized device-vs-oracle parity sweep (development aid; a small fixed
slice runs in tests/test_gpu_fuzz.py).

Each case draws a code (N = 2..4096, k, CRC none/8/16/24), a channel point,
a batch size and decoder knobs, then checks
* SCL (all knobs, DA masks): winners, CRC flags bit-identical to the oracle,
  except frames whose reference winner passes an info position with an fp64
  leaf LLR below fp32 resolution (1e-5, or 4 ulps of the fp32 path metric:
  `precision_limited`) or whose reference list selection kept and dropped
  candidates closer than an fp32 metric can resolve (`selection_limited`);
* BP (crc / reencode / none stop): flags, iterations and u_hat identical on
  all but certified near-tie frames (a small fraction; reported).

    python tests/parity/fuzz_parity.py [cases] [seed]
"""
from __future__ import annotations

import sys

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1609_09358_b200 import BpConfig, CodeConfig, SclConfig, bp_decode_batch, scl_decode_batch  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame  # noqa: E402
from paper_1609_09358_b200.scl import decision_aided_mask  # noqa: E402


def draw_code(rng):
    n = int(rng.integers(1, 13))
    N = 1 << n
    crc = rng.choice([None, 8, 16, 24]) if N >= 32 else None
    lo = (int(crc) + 1) if crc is not None else 1
    if lo > N:
        crc, lo = None, 1
    k = int(rng.integers(lo, N + 1))
    return CodeConfig(N, k, crc=None if crc is None else int(crc))


def frames(code, eb, B, seed):
    sigma = ebno_to_sigma(eb, code.rate)
    x = np.array([make_frame(code, sigma, frame_rng(seed, code.N, f))[1] for f in range(B)])
    return x.astype(np.float32).astype(np.float64)


def _fex(a, b):
    return np.logaddexp(0, a + b) - np.logaddexp(a, b)


def sc_leaf_llrs(llr, u, exact_f):
    """fp64 leaf LLRs along the decision vector u (teacher-forced SC recursion)."""
    out = np.zeros(len(llr))

    def rec(lv, uu, off):
        if len(lv) == 1:
            out[off] = lv[0]
            return np.array([uu[0]])
        h = len(lv) // 2
        a, b = lv[:h], lv[h:]
        f = _fex(a, b) if exact_f else np.sign(a) * np.sign(b) * np.minimum(abs(a), abs(b))
        x1 = rec(f, uu[:h], off)
        x2 = rec(b + (1 - 2 * x1) * a, uu[h:], off + h)
        return np.concatenate([x1 ^ x2, x2])

    rec(np.asarray(llr, dtype=np.float64), np.asarray(u, dtype=np.int64), 0)
    return out


def precision_limited(llr, code, u_ref, exact_f, metric_ref=0.0):
    """The reference's winner passes an info position whose fp64 leaf LLR is
    below fp32 resolution: below 1e-5 (exact-f chains of high-rate codes reach
    0, rounding noise in fp64 itself), or below 4 ulps of the fp32 path metric
    (the two children's metrics differ by |leaf LLR|, so a smaller margin
    cannot be resolved by an fp32 metric of that size)."""
    tol = max(1e-5, 4.0 * float(np.spacing(np.float32(abs(metric_ref)))))
    leaves = sc_leaf_llrs(llr, u_ref, exact_f)
    return bool(np.abs(leaves[np.asarray(code.info_positions)]).min() < tol)


def selection_limited(llr, code, L, da, cfg):
    """A list selection of the reference had its worst kept and best dropped
    candidates closer than the worst-case rounding of an fp32 metric summed
    over that many leaves (0.5 ulp per addition): the fp32 device cannot
    resolve which one the list keeps, so the lists (and possibly the winner)
    part there."""
    gap, metric, leaf = oracle.scl_min_margin(llr, code, L, da=da, metric_mode=cfg.metric_mode, f_mode=cfg.f_mode,
                                              selector=cfg.selector)
    return leaf >= 0 and gap < 0.5 * (leaf + 1) * float(np.spacing(np.float32(abs(metric))))


SCL_CERTIFIED = 0
SCL_FRAMES = 0


def scl_case(rng, seed):
    code = draw_code(rng)
    L = int(rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 20, 32]))  # any list size (N >= 64 if not a power of two)
    if L & (L - 1) and code.N < 64:
        L = 1 << (L.bit_length() - 1)
    cfg = SclConfig(L, metric_mode=str(rng.choice(["exact", "approx"])), f_mode=str(rng.choice(["minsum", "exact"])),
                    selector=str(rng.choice(["pseudo", "bitonic"])),
                    da_threshold=float(rng.choice([0.0, 0.0, 0.3])))
    B = int(rng.integers(1, 40 if code.N <= 1024 else 8))
    eb = float(rng.uniform(-1.0, 4.0))
    llrs = frames(code, eb, B, seed)
    got = scl_decode_batch(llrs, code, cfg)
    da = decision_aided_mask(code, cfg.da_threshold) if cfg.da_threshold > 0 else None
    bad = []
    global SCL_CERTIFIED, SCL_FRAMES
    SCL_FRAMES += B
    for f in range(B):
        ref = oracle.scl_decode(llrs[f], code, L, da=da, metric_mode=cfg.metric_mode, f_mode=cfg.f_mode,
                                selector=cfg.selector)
        if not (np.array_equal(got.u_hat[f], ref["u_hat"]) and bool(got.crc_ok[f]) == ref["crc_ok"]):
            if precision_limited(llrs[f], code, ref["u_hat"], cfg.f_mode == "exact", ref["metric"]) or \
                    selection_limited(llrs[f], code, L, da, cfg):
                SCL_CERTIFIED += 1
            else:
                bad.append(f)
                leaves = sc_leaf_llrs(llrs[f], ref["u_hat"], cfg.f_mode == "exact")
                print(f"  frame {f}: min |fp64 leaf| on info = {np.abs(leaves[np.asarray(code.info_positions)]).min():.3e}, "
                      f"metric dev {float(got.metric[f]):.6f} ref {ref['metric']:.6f}", flush=True)
    return (f"SCL N={code.N} k={code.k} crc={code.crc.width if code.crc else None} {cfg} B={B} eb={eb!r} "
            f"frame_seed={seed}"), bad, B


def bp_case(rng, seed):
    code = draw_code(rng)
    if code.N < 2:
        code = CodeConfig(2, 1)
    mode = str(rng.choice(["crc", "reencode", "none"])) if code.crc is not None else str(
        rng.choice(["reencode", "none"]))
    g_mode = str(rng.choice(["exact", "exact", "min"]))
    i_max = int(rng.integers(1, 40))
    B = int(rng.integers(1, 64 if code.N <= 1024 else 12))
    llrs = frames(code, float(rng.uniform(0.0, 4.0)), B, seed)
    got = bp_decode_batch(llrs, code, BpConfig(i_max=i_max, g_mode=g_mode, stop_mode=mode))
    ref_u, ref_it, ref_cv = oracle.bp_batch(llrs, code, i_max=i_max, g_mode=g_mode, stop_mode=mode)
    same = (got.iterations_used == ref_it) & (got.converged == ref_cv)
    same &= np.array([not ref_cv[f] or np.array_equal(got.u_hat[f], ref_u[f]) for f in range(B)])
    return f"BP N={code.N} k={code.k} {mode} {g_mode} i_max={i_max} B={B}", list(np.flatnonzero(~same)), B


def run(cases=200, seed=1, verbose=True):
    rng = np.random.default_rng(seed)
    fails, scl_bad, bp_diff, bp_frames = [], 0, 0, 0
    for c in range(cases):
        kind = scl_case if c % 2 == 0 else bp_case
        desc, bad, B = kind(rng, seed * 100003 + c)
        if kind is scl_case and bad:
            scl_bad += len(bad)
            fails.append((desc, bad))
        if kind is bp_case:
            bp_diff += len(bad)
            bp_frames += B
        if verbose:
            print(("FAIL " if (bad and kind is scl_case) else ("diff " if bad else "ok   ")) + desc, bad[:5],
                  flush=True)
    return fails, scl_bad, bp_diff, bp_frames


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    s = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    fails, scl_bad, bp_diff, bp_frames = run(n, s)
    print(f"SCL frames differing: {scl_bad}; certified precision-limited: {SCL_CERTIFIED}/{SCL_FRAMES}; "
          f"BP frames differing (near-tie class): {bp_diff}/{bp_frames}")
    sys.exit(1 if fails else 0)
