"""Belief-propagation decoding (reference ``bp.py``), executed by the K1 kernel.

Public surface kept from the reference (``bp.py:27-37``): ``BpConfig``,
``BpGraph``, ``BpResult``, ``g_fn``, ``pe_endpoints``, ``init_graph``,
``iterate_once``, ``stopping_check``, ``bp_decode``.  New: ``bp_decode_batch``
(the batched device entry point the hybrid uses).

Where the work happens:

* ``bp_decode`` / ``bp_decode_batch`` -> ``pc_bp_decode`` (sm_100a K1, fp32,
  CRC / re-encode stop fused, evaluated after every iteration);
* ``iterate_once`` -> ``pc_bp_iterate`` (one device iteration on the given
  graph state, the teacher-forced parity hook);
* ``g_fn``, ``pe_endpoints``, ``init_graph``, ``stopping_check`` are host-side
  helpers on numpy state, as in the reference.

Device arithmetic is fp32: messages agree with the fp64 reference to the
tolerance stated in tests/test_gpu_bp.py; see DESIGN.md "Numerics".
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .channel import LLR_MAX
from .codes import CodeConfig, crc_check, extract_message, polar_transform

__all__ = [
    "BpConfig",
    "BpGraph",
    "BpResult",
    "BpBatchResult",
    "g_fn",
    "pe_endpoints",
    "init_graph",
    "iterate_once",
    "stopping_check",
    "bp_decode",
    "bp_decode_batch",
]

_G_MODES = ("exact", "min")
_STOP_MODES = ("crc", "reencode", "none")


@dataclass(frozen=True)
class BpConfig:
    """Iteration cap, node update, clip bound, stop rule (reference bp.py:40-57)."""

    i_max: int = 50
    g_mode: str = "exact"
    llr_max: float = LLR_MAX
    stop_mode: str = "reencode"

    def __post_init__(self):
        if self.i_max < 1:
            raise ValueError(f"need at least one iteration, got i_max={self.i_max}")
        if self.g_mode not in _G_MODES:
            raise ValueError(f"unknown g mode {self.g_mode!r}")
        if self.llr_max <= 0:
            raise ValueError("clip bound must be positive")
        if self.stop_mode not in _STOP_MODES:
            raise ValueError(f"unknown stop mode {self.stop_mode!r}")

    def native(self, threads_per_frame: int = 0, kernel: int | None = None) -> nat.PcBpCfg:
        return nat.PcBpCfg(
            self.i_max,
            _G_MODES.index(self.g_mode) or (3 if nat.env_int("PC_BP_LOGDOMAIN", 0) else 0),
            _STOP_MODES.index(self.stop_mode),
            threads_per_frame or nat.env_int("PC_BP_TPF", 0),
            float(self.llr_max),
            nat.env_int("PC_BP_KERNEL", 0) if kernel is None else kernel,
        )


@dataclass
class BpGraph:
    """Message state: (n+1, N) arrays, row s = stage s (0 = u side)."""

    l_msgs: np.ndarray
    r_msgs: np.ndarray

    @property
    def n(self) -> int:
        return self.l_msgs.shape[0] - 1

    @property
    def N(self) -> int:
        return self.l_msgs.shape[1]


@dataclass
class BpResult:
    u_hat: np.ndarray
    x_hat: np.ndarray
    soft_u: np.ndarray
    soft_x: np.ndarray
    converged: bool
    iterations_used: int


@dataclass
class BpBatchResult:
    """Batched K1 output.  Arrays are numpy when the input was numpy, else
    device tensors."""

    u_hat: object
    converged: object
    iterations_used: object
    soft_u: object = None
    soft_x: object = None
    payload_words: object = None


def g_fn(a, b, mode: str = "exact", llr_max: float = LLR_MAX):
    """Host form of the node update ln((1+e^(a+b))/(e^a+e^b)), clipped (bp.py:86-100)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if mode == "exact":
        v = np.logaddexp(0.0, a + b) - np.logaddexp(a, b)
    elif mode == "min":
        v = np.sign(a) * np.sign(b) * np.minimum(np.abs(a), np.abs(b))
    else:
        raise ValueError(f"unknown g mode {mode!r}")
    return np.clip(v, -llr_max, llr_max)


def pe_endpoints(j: int, p: int) -> tuple[int, int]:
    """Nodes (i1, i2) joined by processing element p at boundary j (bp.py:103-117)."""
    if j < 1:
        raise ValueError(f"stage boundary starts at 1, got {j}")
    if p < 0:
        raise ValueError(f"element index must be non-negative, got {p}")
    span = 1 << (j - 1)
    i1 = (p >> (j - 1)) * 2 * span + (p & (span - 1))
    return i1, i1 + span


def init_graph(llrs: np.ndarray, code: CodeConfig, cfg: BpConfig) -> BpGraph:
    """L[n] = clip(llr), R[0] = llr_max * frozen, zero elsewhere (bp.py:120-135)."""
    llrs = np.asarray(llrs, dtype=np.float64)
    if llrs.shape != (code.N,):
        raise ValueError(f"expected {code.N} channel LLRs, got shape {llrs.shape}")
    L = np.zeros((code.n + 1, code.N))
    R = np.zeros((code.n + 1, code.N))
    L[code.n] = np.clip(llrs, -cfg.llr_max, cfg.llr_max)
    R[0] = cfg.llr_max * code.frozen_mask
    return BpGraph(l_msgs=L, r_msgs=R)


def iterate_once(graph: BpGraph, code: CodeConfig, cfg: BpConfig) -> BpGraph:
    """One R sweep + L sweep, run on the device (pc_bp_iterate), written back in place."""
    torch = nat.require_device()
    lib = nat.load()
    dc = nat.device_code(code)
    Ld = torch.from_numpy(np.ascontiguousarray(graph.l_msgs, dtype=np.float32)).cuda()
    Rd = torch.from_numpy(np.ascontiguousarray(graph.r_msgs, dtype=np.float32)).cuda()
    ncfg = cfg.native()
    nat.check(
        lib.pc_bp_iterate(nat.ptr(Ld), nat.ptr(Rd), 1, dc.ref, C_byref(ncfg), nat.stream_handle()),
        "pc_bp_iterate",
    )
    graph.l_msgs[...] = Ld.cpu().numpy().astype(np.float64)
    graph.r_msgs[...] = Rd.cpu().numpy().astype(np.float64)
    return graph


def C_byref(x):
    import ctypes

    return ctypes.byref(x)


def _hard(soft: np.ndarray) -> np.ndarray:
    return (soft < 0).astype(np.uint8)  # an exact 0 decides bit 0


def stopping_check(graph: BpGraph, code: CodeConfig, cfg: BpConfig) -> bool:
    """Host evaluation of the stop rule on explicit state (bp.py:176-191)."""
    if cfg.stop_mode == "none":
        return False
    n = graph.n
    u_hat = _hard(graph.l_msgs[0] + graph.r_msgs[0])
    if cfg.stop_mode == "reencode":
        return bool(np.array_equal(polar_transform(u_hat), _hard(graph.l_msgs[n] + graph.r_msgs[n])))
    if code.crc is None:
        raise ValueError("crc stop mode needs a code with a CRC")
    return crc_check(extract_message(u_hat, code), code.crc)


def _validate_cfg(code: CodeConfig, cfg: BpConfig):
    if code.N < 2:
        raise ValueError("decoding needs a block length of at least 2")
    if cfg.stop_mode == "crc" and code.crc is None:
        raise ValueError("crc stop mode needs a code with a CRC")


def bp_decode_batch(
    llrs,
    code: CodeConfig,
    cfg: BpConfig | None = None,
    *,
    soft: bool = False,
    payload: bool = False,
    stream=None,
) -> BpBatchResult:
    """Decode B frames ``llrs[B, N]`` with one K1 launch.

    ``llrs`` may be a numpy array (copied to the device, results returned as
    numpy) or a CUDA tensor (results stay on the device).
    """
    cfg = cfg or BpConfig()
    _validate_cfg(code, cfg)
    torch = nat.require_device()
    lib = nat.load()
    host = not (hasattr(llrs, "is_cuda") and llrs.is_cuda)
    if host:
        arr = np.asarray(llrs, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[1] != code.N:
            raise ValueError(f"expected llrs of shape (B, {code.N}), got {arr.shape}")
        x = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).cuda()
    else:
        if llrs.dim() != 2 or llrs.shape[1] != code.N:
            raise ValueError(f"expected llrs of shape (B, {code.N}), got {tuple(llrs.shape)}")
        x = llrs.to(torch.float32).contiguous()
    B = x.shape[0]
    dev = x.device
    NW = (code.N + 31) // 32
    MW = (code.message_len + 31) // 32
    cur = torch.cuda.current_stream(dev)
    u = torch.empty((B, NW), dtype=torch.int32, device=dev)
    it = torch.empty(B, dtype=torch.int32, device=dev)
    cv = torch.empty(B, dtype=torch.uint8, device=dev)
    su = torch.empty((B, code.N), dtype=torch.float32, device=dev) if soft else None
    sx = torch.empty((B, code.N), dtype=torch.float32, device=dev) if soft else None
    pw = torch.empty((B, MW), dtype=torch.int32, device=dev) if payload else None
    dc = nat.device_code(code)
    ncfg = cfg.native()
    wk = torch.empty(1, dtype=torch.int32, device=dev)  # frame counter of the persistent kernel (small N)
    ncfg.work = wk.data_ptr()
    if stream is not None:  # the launch stream sees the input converted on the current stream
        stream.wait_stream(cur)
    nat.check(
        lib.pc_bp_decode(
            nat.ptr(x), B, dc.ref, C_byref(ncfg), nat.ptr(u), nat.ptr(pw), nat.ptr(su), nat.ptr(sx),
            nat.ptr(it), nat.ptr(cv), None, nat.stream_handle(stream),
        ),
        "pc_bp_decode",
    )
    if stream is not None:  # results are read on the current stream; temporaries outlive the launch
        for t in (x, u, it, cv, su, sx, pw, wk):
            if t is not None:
                t.record_stream(stream)
        cur.wait_stream(stream)
    if not host:
        return BpBatchResult(u, cv.bool(), it, su, sx, pw)
    ub = nat.unpack_bits(u.cpu().numpy().view(np.uint32), code.N)
    return BpBatchResult(
        u_hat=ub,
        converged=cv.cpu().numpy().astype(bool),
        iterations_used=it.cpu().numpy().astype(np.int64),
        soft_u=None if su is None else su.cpu().numpy().astype(np.float64),
        soft_x=None if sx is None else sx.cpu().numpy().astype(np.float64),
        payload_words=None if pw is None else pw.cpu().numpy().view(np.uint32),
    )


def bp_decode(llrs: np.ndarray, code: CodeConfig, cfg: BpConfig | None = None) -> BpResult:
    """Decode one frame on the device (reference bp.py:194-217)."""
    cfg = cfg or BpConfig()
    _validate_cfg(code, cfg)
    llrs = np.asarray(llrs, dtype=np.float64)
    if llrs.shape != (code.N,):
        raise ValueError(f"expected {code.N} channel LLRs, got shape {llrs.shape}")
    r = bp_decode_batch(llrs[None, :], code, cfg, soft=True)
    su, sx = r.soft_u[0], r.soft_x[0]
    return BpResult(
        u_hat=r.u_hat[0].copy(),  # the kernel's own decisions (the batch API's u_hat)
        x_hat=_hard(sx),
        soft_u=su,
        soft_x=sx,
        converged=bool(r.converged[0]),
        iterations_used=int(r.iterations_used[0]),
    )
