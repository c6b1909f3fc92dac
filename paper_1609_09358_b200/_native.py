"""ctypes binding of ``libpolarcuda.so`` (include/polarcuda.h) plus device tables.

The shared library is built in-tree by ``csrc/Makefile`` (``__graft_entry__.build``).
PyTorch only provides device memory, streams and events here; every decode
runs in the hand-written sm_100a kernels behind the C-ABI.  There is no CPU
fallback: without the library or without a B200 the calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
from collections import OrderedDict
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libpolarcuda.so"

PC_OK = 0

EXPORTS = (
    "pc_version",
    "pc_strerror",
    "pc_code_seal",
    "pc_workspace_bytes",
    "pc_device_count",
    "pc_bp_decode",
    "pc_bp_iterate",
    "pc_compact",
    "pc_scl_decode",
    "pc_scl_workspace_bytes",
    "pc_encode",
    "pc_gen_frames",
    "pc_count_errors",
    "pc_stamp",
)


class PcCode(C.Structure):
    _fields_ = [
        ("N", C.c_int32),
        ("n", C.c_int32),
        ("k", C.c_int32),
        ("m", C.c_int32),
        ("crc_width", C.c_int32),
        ("crc_offset", C.c_uint32),
        ("enc_crc_offset", C.c_uint32),
        ("first_info", C.c_int32),
        ("frozen_bits", C.c_void_p),
        ("crc_cols", C.c_void_p),
        ("info_pos", C.c_void_p),
        ("enc_cols", C.c_void_p),
        ("da_bits", C.c_void_p),
        ("seal", C.c_uint64),
    ]


class PcBpCfg(C.Structure):
    _fields_ = [
        ("i_max", C.c_int32),
        ("g_mode", C.c_int32),
        ("stop_mode", C.c_int32),
        ("threads_per_frame", C.c_int32),
        ("llr_max", C.c_float),
        ("kernel", C.c_int32),
        ("work", C.c_void_p),
    ]


class PcSclCfg(C.Structure):
    _fields_ = [
        ("L", C.c_int32),
        ("metric_exact", C.c_int32),
        ("f_exact", C.c_int32),
        ("selector_bitonic", C.c_int32),
        ("virtual_levels", C.c_int32),
        ("warps_per_cta", C.c_int32),
        ("kernel", C.c_int32),
    ]


class NativeUnavailable(RuntimeError):
    """The CUDA library or a B200 is missing; there is no CPU fallback."""


_lib = None


def load():
    """Load the C-ABI library (no device needed to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = C.CDLL(str(LIB_PATH))
    vp, i32, i64, u64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_float
    sig = {
        "pc_version": (i32, []),
        "pc_strerror": (C.c_char_p, [i32]),
        "pc_code_seal": (i32, [vp, vp]),
        "pc_workspace_bytes": (i64, []),
        "pc_device_count": (i32, []),
        "pc_bp_decode": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "pc_bp_iterate": (i32, [vp, vp, i32, vp, vp, vp]),
        "pc_compact": (i32, [vp, i32, vp, vp, vp, vp]),
        "pc_scl_decode": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "pc_scl_workspace_bytes": (i64, [vp, vp]),
        "pc_encode": (i32, [vp, i32, vp, vp, vp]),
        "pc_gen_frames": (i32, [u64, i32, i64, i32, f32, vp, vp, vp, vp]),
        "pc_count_errors": (i32, [vp, vp, i32, i32, vp, vp]),
        "pc_stamp": (i32, [vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != PC_OK:
        msg = load().pc_strerror(rc).decode()
        raise RuntimeError(f"{what} failed: {msg} (code {rc})")


def require_device():
    """Return torch after checking a B200 and the library; raise otherwise."""
    import torch

    lib = load()
    if not torch.cuda.is_available() or lib.pc_device_count() < 1:
        raise NativeUnavailable("no sm_100 CUDA device visible; the decoders have no CPU fallback")
    return torch


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """[..., L] 0/1 -> [..., ceil(L/32)] uint32, bit b at word b//32 position b%32."""
    bits = np.asarray(bits, dtype=np.uint8)
    L = bits.shape[-1]
    W = (L + 31) // 32
    pad = np.zeros(bits.shape[:-1] + (W * 32,), dtype=np.uint8)
    pad[..., :L] = bits
    b = pad.reshape(*bits.shape[:-1], W, 32).astype(np.uint32)
    return (b << np.arange(32, dtype=np.uint32)).sum(axis=-1, dtype=np.uint64).astype(np.uint32)


def unpack_bits(words: np.ndarray, L: int) -> np.ndarray:
    w = np.asarray(words, dtype=np.uint32)
    bits = (w[..., :, None] >> np.arange(32, dtype=np.uint32)) & 1
    return bits.reshape(*w.shape[:-1], w.shape[-1] * 32)[..., :L].astype(np.uint8)


class DeviceCode:
    """Device-resident tables of a CodeConfig plus the pc_code_t struct."""

    def __init__(self, code, device=None, da_mask=None):
        torch = require_device()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.code = code
        self.device = dev
        cols, off = code.crc_columns()
        ecols, eoff = code.encoder_columns()

        def t(a, dtype):
            return torch.from_numpy(np.ascontiguousarray(a).astype(dtype, copy=False)).to(dev)

        self.frozen_bits = t(pack_bits(code.frozen_mask).view(np.int32), np.int32)
        self.crc_cols = t(cols.view(np.int32), np.int32)
        self.info_pos = t(code.info_positions.astype(np.int32), np.int32)
        self.enc_cols = t((ecols if ecols.size else np.zeros(1, np.uint32)).view(np.int32), np.int32)
        self.da_bits = None
        if da_mask is not None and np.any(da_mask):
            self.da_bits = t(pack_bits(np.asarray(da_mask, np.uint8)).view(np.int32), np.int32)
        self.struct = PcCode(
            code.N,
            code.n,
            code.k,
            code.message_len,
            code.crc_width,
            off,
            eoff,
            0,  # first_info: derived by pc_code_seal
            ptr(self.frozen_bits),
            ptr(self.crc_cols),
            ptr(self.info_pos),
            ptr(self.enc_cols),
            ptr(self.da_bits),
        )
        # the library validates the device tables, derives first_info and seals the struct
        check(load().pc_code_seal(C.byref(self.struct), stream_handle()), "pc_code_seal")
        self.workspace = torch.zeros(max(1, load().pc_workspace_bytes() // 4), dtype=torch.int32, device=dev)

    @property
    def ref(self):
        return C.byref(self.struct)

    def scl_workspace_bytes(self, ncfg) -> int:
        nbytes = int(load().pc_scl_workspace_bytes(self.ref, C.byref(ncfg)))
        if nbytes < 0:
            raise RuntimeError("pc_scl_workspace_bytes rejected the configuration")
        return nbytes

    def new_scl_workspace(self, ncfg, stream=None):
        """A workspace private to one caller (torch caching allocator; recorded
        on ``stream`` so it is not reused before that stream's launch ends)."""
        import torch

        ws = torch.empty((self.scl_workspace_bytes(ncfg) + 3) // 4, dtype=torch.int32, device=self.device)
        if stream is not None:
            ws.record_stream(stream)
        return ws

    def scl_workspace(self, ncfg):
        """Device workspace for pc_scl_decode with this code and PcSclCfg (cached
        by size and shared: for callers that order their launches on one stream)."""
        import torch

        nbytes = int(load().pc_scl_workspace_bytes(self.ref, C.byref(ncfg)))
        if nbytes < 0:
            raise RuntimeError("pc_scl_workspace_bytes rejected the configuration")
        ws = getattr(self, "_scl_ws", None)
        if ws is None or ws.numel() * 4 < nbytes:
            ws = torch.zeros((nbytes + 3) // 4, dtype=torch.int32, device=self.device)
            self._scl_ws = ws
        return ws

    def with_da(self, da_mask):
        """Same code with a decision-aided position mask (SclConfig.da_threshold)."""
        if da_mask is None or not np.any(da_mask):
            return self
        return DeviceCode(self.code, self.device, da_mask)


_CODE_CACHE: "OrderedDict" = OrderedDict()
_CODE_CACHE_MAX = 16  # device tables of the most recently used codes (a sweep builds a CodeConfig per point)


def _cached(key, code, make):
    dc = _CODE_CACHE.get(key)
    if dc is None or dc.code is not code:  # (an id() reused by a new CodeConfig is a miss)
        dc = make()
        _CODE_CACHE[key] = dc
    _CODE_CACHE.move_to_end(key)
    while len(_CODE_CACHE) > _CODE_CACHE_MAX:
        _CODE_CACHE.popitem(last=False)  # holders (decoders) keep their own reference
    return dc


def device_code(code, da_mask=None) -> DeviceCode:
    import torch

    key = (id(code), torch.cuda.current_device())
    dc = _cached(key, code, lambda: DeviceCode(code))
    if da_mask is not None and np.any(da_mask):
        dkey = key + (pack_bits(np.asarray(da_mask, np.uint8)).tobytes(),)
        return _cached(dkey, code, lambda: DeviceCode(code, dc.device, da_mask))
    return dc


def env_int(name: str, default: int) -> int:
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default
