"""CPU parity oracle (TEST INFRASTRUCTURE -- never on the product path).

ctypes front-end for ``oracle/liboracle.so`` (built from ``oracle/oracle.c``
by ``oracle/Makefile``), a plain-C fp64 restatement of the reference
``polarsim`` decoders.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
CPU legs of ``bench.py`` may import this package.

Functions take a ``CodeConfig`` from ``paper_1609_09358_b200`` (pure host
description, no device state) and numpy arrays.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None


class _OcCode(C.Structure):
    _fields_ = [
        ("N", C.c_int32),
        ("n", C.c_int32),
        ("k", C.c_int32),
        ("m", C.c_int32),
        ("frozen", C.c_void_p),
        ("info_pos", C.c_void_p),
        ("crc_width", C.c_int32),
        ("crc_poly", C.c_uint32),
        ("crc_init", C.c_uint32),
    ]


def build(force: bool = False) -> Path:
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < (_HERE / "oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(_LIB_PATH))
        vp, i32, f64, u32 = C.c_void_p, C.c_int32, C.c_double, C.c_uint32
        sig = {
            "oc_bp_iterate": (None, [vp, vp, i32, i32, i32, f64]),
            "oc_bp_decode": (i32, [vp, vp, i32, i32, f64, i32, vp, vp, vp, vp, vp]),
            "oc_bp_g": (f64, [f64, f64, i32, f64]),
            "oc_scl_paths": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, vp, vp]),
            "oc_set_margin_out": (None, [vp]),
            "oc_scl_decode": (i32, [vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, vp]),
            "oc_scl_f": (f64, [f64, f64, i32]),
            "oc_metric_inc": (f64, [f64, i32, i32]),
            "oc_select_keep": (i32, [vp, i32, i32, i32, vp]),
            "oc_hybrid_frame": (i32, [vp, vp, i32, i32, f64, i32, i32, i32, vp, vp, vp]),
            "oc_bp_batch": (i32, [vp, i32, vp, i32, i32, f64, i32, vp, vp, vp, i32]),
            "oc_scl_batch": (i32, [vp, i32, vp, vp, i32, i32, i32, vp, vp, vp, i32]),
            "oc_hybrid_batch": (i32, [vp, i32, vp, i32, i32, f64, i32, i32, i32, vp, vp, vp, i32]),
            "oc_polar_transform": (None, [vp, i32]),
            "oc_encode": (None, [vp, vp, vp]),
            "oc_crc_register_bits": (u32, [vp, i32, i32, u32, u32]),
            "oc_max_threads": (i32, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OracleCode:
    """Keeps the numpy buffers alive behind the C struct."""

    def __init__(self, code):
        self.code = code
        self.frozen = np.ascontiguousarray(code.frozen_mask, dtype=np.uint8)
        self.info = np.ascontiguousarray(code.info_positions, dtype=np.int32)
        crc = code.crc
        self.s = _OcCode(
            code.N,
            code.n,
            code.k,
            code.message_len,
            self.frozen.ctypes.data,
            self.info.ctypes.data,
            0 if crc is None else crc.width,
            0 if crc is None else crc.poly,
            0 if crc is None else crc.init,
        )

    @property
    def ref(self):
        return C.byref(self.s)


_CODES: dict = {}


def _oc(code) -> OracleCode:
    key = id(code)
    oc = _CODES.get(key)
    if oc is None or oc.code is not code:
        oc = OracleCode(code)
        _CODES[key] = oc
    return oc


_STOP = {"crc": 0, "reencode": 1, "none": 2}


def bp_iterate(l_msgs: np.ndarray, r_msgs: np.ndarray, g_mode="exact", llr_max=20.0):
    """One iterate_once on copies of fp64 (n+1, N) arrays (reference bp.py:138-161)."""
    L = np.array(l_msgs, dtype=np.float64, order="C", copy=True)
    R = np.array(r_msgs, dtype=np.float64, order="C", copy=True)
    n = L.shape[0] - 1
    lib().oc_bp_iterate(_p(L), _p(R), n, L.shape[1], int(g_mode == "exact"), float(llr_max))
    return L, R


def bp_g(a: float, b: float, g_mode="exact", llr_max=20.0) -> float:
    return lib().oc_bp_g(float(a), float(b), int(g_mode == "exact"), float(llr_max))


def bp_decode(llrs, code, i_max=50, g_mode="exact", llr_max=20.0, stop_mode="reencode"):
    """fp64 bp_decode (reference bp.py:194-217) -> dict."""
    llrs = np.ascontiguousarray(llrs, dtype=np.float64)
    u = np.zeros(code.N, np.uint8)
    su = np.zeros(code.N)
    sx = np.zeros(code.N)
    it = np.zeros(1, np.int32)
    cv = np.zeros(1, np.uint8)
    rc = lib().oc_bp_decode(
        _p(llrs), _oc(code).ref, i_max, int(g_mode == "exact"), llr_max, _STOP[stop_mode],
        _p(u), _p(su), _p(sx), _p(it), _p(cv),
    )
    if rc:
        raise ValueError("oracle bp_decode rejected its arguments")
    return dict(u_hat=u, soft_u=su, soft_x=sx, iterations_used=int(it[0]), converged=bool(cv[0]))


def scl_paths(llrs, code, L, da=None, metric_mode="exact", f_mode="minsum", selector="pseudo"):
    llrs = np.ascontiguousarray(llrs, dtype=np.float64)
    da = np.zeros(code.N, np.uint8) if da is None else np.ascontiguousarray(da, dtype=np.uint8)
    up = np.zeros((L, code.N), np.uint8)
    mt = np.zeros(L)
    P = lib().oc_scl_paths(
        _p(llrs), _p(_oc(code).frozen), _p(da), code.N, L, int(metric_mode == "exact"),
        int(f_mode == "exact"), int(selector == "bitonic"), _p(up), _p(mt),
    )
    return up[:P], mt[:P]


def scl_decode(llrs, code, L, da=None, metric_mode="exact", f_mode="minsum", selector="pseudo"):
    """Winner of the reference list decoder (reference scl.py:151-197) -> dict."""
    llrs = np.ascontiguousarray(llrs, dtype=np.float64)
    da_arr = None if da is None else np.ascontiguousarray(da, dtype=np.uint8)
    u = np.zeros(code.N, np.uint8)
    mt = np.zeros(1)
    ok = np.zeros(1, np.uint8)
    sel = np.zeros(1, np.uint8)
    P = lib().oc_scl_decode(
        _p(llrs), _oc(code).ref, None if da_arr is None else _p(da_arr), L, int(metric_mode == "exact"),
        int(f_mode == "exact"), int(selector == "bitonic"), _p(u), _p(mt), _p(ok), _p(sel),
    )
    if P < 0:
        raise ValueError("oracle scl_decode rejected its arguments")
    return dict(u_hat=u, metric=float(mt[0]), crc_ok=bool(ok[0]), selected_by_crc=bool(sel[0]), paths=P)


def scl_f(a, b, exact=False):
    return lib().oc_scl_f(float(a), float(b), int(exact))


def metric_inc(lam, u, exact=True):
    return lib().oc_metric_inc(float(lam), int(u), int(exact))


def select_keep(cand, L, bitonic=False):
    cand = np.ascontiguousarray(cand, dtype=np.float64)
    keep = np.zeros(cand.size, np.uint8)
    lib().oc_select_keep(_p(cand), cand.size, L, int(bitonic), _p(keep))
    return keep


def hybrid_frame(llrs, code, i_max=50, g_mode="exact", llr_max=20.0, L=32, metric_mode="exact", f_mode="minsum"):
    llrs = np.ascontiguousarray(llrs, dtype=np.float64)
    pay = np.zeros(code.message_len, np.uint8)
    prov = np.zeros(1, np.uint8)
    it = np.zeros(1, np.int32)
    rc = lib().oc_hybrid_frame(
        _p(llrs), _oc(code).ref, i_max, int(g_mode == "exact"), llr_max, L, int(metric_mode == "exact"),
        int(f_mode == "exact"), _p(pay), _p(prov), _p(it),
    )
    if rc:
        raise ValueError("oracle hybrid rejected its arguments")
    return pay, ("scl" if prov[0] else "bp"), int(it[0])


def bp_batch(llrs, code, i_max=50, g_mode="exact", llr_max=20.0, stop_mode="crc", nthreads=0):
    llrs = np.ascontiguousarray(llrs, dtype=np.float64)
    B = llrs.shape[0]
    u = np.zeros((B, code.N), np.uint8)
    it = np.zeros(B, np.int32)
    cv = np.zeros(B, np.uint8)
    rc = lib().oc_bp_batch(
        _p(llrs), B, _oc(code).ref, i_max, int(g_mode == "exact"), llr_max, _STOP[stop_mode],
        _p(u), _p(it), _p(cv), nthreads,
    )
    if rc:
        raise ValueError("oracle bp_batch failed")
    return u, it, cv.astype(bool)


def scl_batch(llrs, code, L, metric_mode="exact", f_mode="minsum", nthreads=0):
    llrs = np.ascontiguousarray(llrs, dtype=np.float64)
    B = llrs.shape[0]
    u = np.zeros((B, code.N), np.uint8)
    mt = np.zeros(B)
    ok = np.zeros(B, np.uint8)
    rc = lib().oc_scl_batch(
        _p(llrs), B, _oc(code).ref, None, L, int(metric_mode == "exact"), int(f_mode == "exact"),
        _p(u), _p(mt), _p(ok), nthreads,
    )
    if rc:
        raise ValueError("oracle scl_batch failed")
    return u, mt, ok.astype(bool)


def hybrid_batch(llrs, code, i_max=50, L=32, g_mode="exact", llr_max=20.0, metric_mode="exact",
                 f_mode="minsum", nthreads=0):
    llrs = np.ascontiguousarray(llrs, dtype=np.float64)
    B = llrs.shape[0]
    pay = np.zeros((B, code.message_len), np.uint8)
    prov = np.zeros(B, np.uint8)
    it = np.zeros(B, np.int32)
    rc = lib().oc_hybrid_batch(
        _p(llrs), B, _oc(code).ref, i_max, int(g_mode == "exact"), llr_max, L, int(metric_mode == "exact"),
        int(f_mode == "exact"), _p(pay), _p(prov), _p(it), nthreads,
    )
    if rc:
        raise ValueError("oracle hybrid_batch failed")
    return pay, prov.astype(bool), it


def polar_transform(u):
    x = np.array(u, dtype=np.uint8, order="C", copy=True)
    lib().oc_polar_transform(_p(x), x.size)
    return x


def encode(msg, code):
    msg = np.ascontiguousarray(msg, dtype=np.uint8)
    x = np.zeros(code.N, np.uint8)
    lib().oc_encode(_p(msg), _oc(code).ref, _p(x))
    return x


def crc_register(bits, width, poly, init=0):
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    return int(lib().oc_crc_register_bits(_p(bits), bits.size, width, poly, init))


def max_threads() -> int:
    return int(lib().oc_max_threads())


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def scl_min_margin(llr, code, L, da=None, metric_mode="exact", f_mode="minsum", selector="pseudo"):
    """(gap, metric, leaf): the smallest gap between the worst kept and the best
    dropped candidate over the frame's list selections (single-threaded; a
    test diagnostic for fp32 selection ties)."""
    out = np.array([np.inf, 0.0, -1.0])
    lib().oc_set_margin_out(_p(out))
    try:
        scl_decode(llr, code, L, da=da, metric_mode=metric_mode, f_mode=f_mode, selector=selector)
    finally:
        lib().oc_set_margin_out(None)
    return float(out[0]), float(out[1]), int(out[2])
