"""CRC-aided successive-cancellation list decoding (reference ``scl.py``).

Public surface kept from the reference (``scl.py:26-36``).  ``scl_decode`` and
the new ``scl_decode_batch`` run the K3 kernel (``pc_scl_decode``); the scalar
helpers (``sc_f``, ``sc_g``, ``path_metric_update``) and the selector
functions are host utilities with the reference's semantics, used by tests
and by callers that reason about single values.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .codes import CodeConfig

__all__ = [
    "SclConfig",
    "SclResult",
    "SclBatchResult",
    "sc_f",
    "sc_g",
    "path_metric_update",
    "pseudo_sort_select",
    "bitonic_sort_select",
    "decision_aided_mask",
    "scl_decode",
    "scl_decode_batch",
]


@dataclass(frozen=True)
class SclConfig:
    """List size and decoder flavour (reference scl.py:39-66)."""

    list_size: int = 8
    metric_mode: str = "exact"
    f_mode: str = "minsum"
    selector: str = "pseudo"
    da_threshold: float = 0.0

    def __post_init__(self):
        if self.list_size < 1:
            raise ValueError(f"list size must be at least 1, got {self.list_size}")
        if self.metric_mode not in ("exact", "approx"):
            raise ValueError(f"unknown metric mode {self.metric_mode!r}")
        if self.f_mode not in ("minsum", "exact"):
            raise ValueError(f"unknown check-node mode {self.f_mode!r}")
        if self.selector not in ("pseudo", "bitonic"):
            raise ValueError(f"unknown selector {self.selector!r}")
        if not 0.0 <= self.da_threshold <= 1.0:
            raise ValueError("decision-aid threshold must lie in [0, 1]")

    def native(self, virtual_levels: int | None = None, warps_per_cta: int = 0, kernel: int | None = None) -> nat.PcSclCfg:
        if self.list_size > 32:
            raise ValueError(f"the device list decoder supports list sizes up to 32, got {self.list_size}")
        return nat.PcSclCfg(
            self.list_size,
            int(self.metric_mode == "exact"),
            int(self.f_mode == "exact"),
            int(self.selector == "bitonic"),
            nat.env_int("PC_SCL_NV", -1) if virtual_levels is None else virtual_levels,
            warps_per_cta or nat.env_int("PC_SCL_WPC", 1),
            nat.env_int("PC_SCL_KERNEL", 0) if kernel is None else kernel,
        )


@dataclass
class SclResult:
    u_hat: np.ndarray
    metric: float
    crc_ok: bool
    selected_by_crc: bool


@dataclass
class SclBatchResult:
    u_hat: object
    metric: object
    crc_ok: object
    selected_by_crc: object
    payload_words: object = None


# ------------------------------------------------------------ scalar helpers --


def _f_min(a: float, b: float) -> float:
    if a == 0.0 or b == 0.0:
        return 0.0
    m = min(abs(a), abs(b))
    return -m if (a < 0.0) != (b < 0.0) else m


def _f_exact(a: float, b: float) -> float:
    s = a + b
    num = s + math.log1p(math.exp(-s)) if s > 0.0 else math.log1p(math.exp(s))
    hi, lo = (a, b) if a >= b else (b, a)
    return num - (hi + math.log1p(math.exp(lo - hi)))


def sc_f(a: float, b: float, exact: bool = False) -> float:
    """Check-node update: min-sum, or exact box-plus (_kernels.py:40-65)."""
    return float(_f_exact(a, b) if exact else _f_min(a, b))


def sc_g(a: float, b: float, u: int) -> float:
    """Variable-node update b + (1 - 2u) a (_kernels.py:68-73)."""
    return float(b - a if u else b + a)


def _inc(lam: float, u: int, exact: bool) -> float:
    x = -lam if u else lam
    if exact:
        return math.log1p(math.exp(-x)) if x > 0.0 else -x + math.log1p(math.exp(x))
    return -x if x < 0.0 else 0.0


def path_metric_update(metric: float, llr: float, u: int, mode: str = "exact") -> float:
    """metric + ln(1 + exp(-(1-2u) llr)) (exact) or |llr| on disagreement (approx)."""
    if mode not in ("exact", "approx"):
        raise ValueError(f"unknown metric mode {mode!r}")
    return metric + float(_inc(float(llr), int(u), mode == "exact"))


def _order_keys(metrics: np.ndarray) -> np.ndarray:
    """Candidate ranks under (metric, index), 1-based (pairwise counting)."""
    m = metrics
    idx = np.arange(m.size)
    before = (m[None, :] < m[:, None]) | ((m[None, :] == m[:, None]) & (idx[None, :] <= idx[:, None]))
    return before.sum(axis=1)


def pseudo_sort_select(metrics: np.ndarray, L: int) -> np.ndarray:
    """Survivors by pairwise ranking, best first; infinities never survive (scl.py:103-117)."""
    m = np.ascontiguousarray(metrics, dtype=np.float64)
    if L < 1:
        raise ValueError("need L >= 1")
    d = _order_keys(m)
    keep = (d <= L) & np.isfinite(m)
    sel = np.flatnonzero(keep)
    return sel[np.argsort(d[sel], kind="stable")]


def _bitonic_network(keys: np.ndarray, idx: np.ndarray) -> None:
    size = keys.size
    k = 2
    while k <= size:
        j = k >> 1
        while j:
            i = np.arange(size)
            partner = i ^ j
            lo = i[partner > i]
            hi = partner[partner > i]
            a, b = keys[lo], keys[hi]
            ia, ib = idx[lo], idx[hi]
            a_after = (a > b) | ((a == b) & (ia > ib))
            b_after = (a < b) | ((a == b) & (ia < ib))
            up = (lo & k) == 0
            swap = (up & a_after) | (~up & b_after)
            keys[lo[swap]], keys[hi[swap]] = b[swap], a[swap]
            idx[lo[swap]], idx[hi[swap]] = ib[swap], ia[swap]
            j >>= 1
        k <<= 1


def bitonic_sort_select(metrics: np.ndarray, L: int) -> np.ndarray:
    """Survivors via a full bitonic network on (metric, index) (scl.py:120-136)."""
    m = np.asarray(metrics, dtype=np.float64)
    if L < 1:
        raise ValueError("need L >= 1")
    size = 1
    while size < max(m.size, 2):
        size <<= 1
    keys = np.full(size, np.inf)
    keys[: m.size] = m
    idx = np.arange(size, dtype=np.int64)
    _bitonic_network(keys, idx)
    return idx[:L][np.isfinite(keys[:L])].copy()


def decision_aided_mask(code: CodeConfig, threshold: float) -> np.ndarray:
    """Non-frozen positions with Bhattacharyya value strictly below threshold (scl.py:139-148)."""
    if not 0.0 <= threshold <= 1.0:
        raise ValueError("decision-aid threshold must lie in [0, 1]")
    return ((code.bhattacharyya < threshold) & (code.frozen_mask == 0)).astype(np.uint8)


# ------------------------------------------------------------ device decode --


def scl_decode_batch(
    llrs,
    code: CodeConfig,
    cfg: SclConfig | None = None,
    *,
    queue=None,
    count=None,
    payload: bool = False,
    stream=None,
) -> SclBatchResult:
    """List-decode ``llrs[B, N]`` (numpy -> numpy results, CUDA tensor -> tensors).

    With ``queue``/``count`` (device int32) only the queued frames are decoded
    and outputs are indexed by frame (the hybrid's use).
    """
    cfg = cfg or SclConfig()
    if code.N < 2:
        raise ValueError("list decoding needs a block length of at least 2")
    L = cfg.list_size
    if L & (L - 1) and code.N < 64:
        raise ValueError(f"a list size that is not a power of two (L={L}) needs N >= 64 on the device")
    torch = nat.require_device()
    lib = nat.load()
    host = not (hasattr(llrs, "is_cuda") and llrs.is_cuda)
    if host:
        arr = np.asarray(llrs, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[1] != code.N:
            raise ValueError(f"expected llrs of shape (B, {code.N}), got {arr.shape}")
        if not np.isfinite(arr).all():
            raise ValueError("channel LLRs must be finite")
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
    if stream is not None:  # the launch stream sees the inputs and zeroed outputs made on the current stream
        stream.wait_stream(cur)
    u = torch.zeros((B, NW), dtype=torch.int32, device=dev)
    mt = torch.zeros(B, dtype=torch.float32, device=dev)
    ok = torch.zeros(B, dtype=torch.uint8, device=dev)
    sel = torch.zeros(B, dtype=torch.uint8, device=dev)
    pw = torch.zeros((B, MW), dtype=torch.int32, device=dev) if payload else None
    da = decision_aided_mask(code, cfg.da_threshold) if cfg.da_threshold > 0 else None
    dc = nat.device_code(code, da)
    ncfg = cfg.native()
    import ctypes

    if stream is not None:
        stream.wait_stream(cur)
    nat.check(
        lib.pc_scl_decode(
            nat.ptr(x), B, nat.ptr(queue), nat.ptr(count), dc.ref, ctypes.byref(ncfg), nat.ptr(u), nat.ptr(pw),
            nat.ptr(mt), nat.ptr(ok), nat.ptr(sel), None, nat.ptr(dc.new_scl_workspace(ncfg, stream)),
            nat.stream_handle(stream),
        ),
        "pc_scl_decode",
    )
    if stream is not None:  # results are read on the current stream; the temporaries outlive the launch
        for t in (x, u, mt, ok, sel, pw, queue, count):
            if t is not None:
                t.record_stream(stream)
        cur.wait_stream(stream)
    if not host:
        return SclBatchResult(u, mt, ok.bool(), sel.bool(), pw)
    return SclBatchResult(
        u_hat=nat.unpack_bits(u.cpu().numpy().view(np.uint32), code.N),
        metric=mt.cpu().numpy().astype(np.float64),
        crc_ok=ok.cpu().numpy().astype(bool),
        selected_by_crc=sel.cpu().numpy().astype(bool),
        payload_words=None if pw is None else pw.cpu().numpy().view(np.uint32),
    )


def scl_decode(llrs: np.ndarray, code: CodeConfig, cfg: SclConfig | None = None) -> SclResult:
    """List-decode one frame on the device (reference scl.py:151-197)."""
    cfg = cfg or SclConfig()
    llrs = np.ascontiguousarray(llrs, dtype=np.float64)
    if llrs.shape != (code.N,):
        raise ValueError(f"expected {code.N} channel LLRs, got shape {llrs.shape}")
    if code.N < 2:
        raise ValueError("list decoding needs a block length of at least 2")
    if not np.isfinite(llrs).all():
        raise ValueError("channel LLRs must be finite")
    r = scl_decode_batch(llrs[None, :], code, cfg)
    return SclResult(
        u_hat=r.u_hat[0].copy(),
        metric=float(r.metric[0]),
        crc_ok=bool(r.crc_ok[0]),
        selected_by_crc=bool(r.selected_by_crc[0]),
    )
