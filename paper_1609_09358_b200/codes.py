"""Polar code description on the host: construction, CRC, bit placement.

This module restates the code-level contract of the reference
(`/root/reference/pkg/src/polarsim/polar.py`) so that every constant the
device kernels consume is bit-exact with it:

* frozen set: Bhattacharyya/BEC doubling recursion, the ``N - k`` least
  reliable positions frozen, ties resolved toward the lower index
  (reference ``polar.py:106-144``);
* CRC: MSB-first shift register, no reflection, no final XOR
  (reference ``polar.py:147-179``);
* placement: payload then CRC remainder at the non-frozen positions in
  ascending order (reference ``polar.py:289-314``).

Beyond the reference API this module derives the *affine GF(2) tables* the
GPU uses instead of clocking a register bit by bit:

* ``crc_columns``: for every block position the CRC-register contribution of
  a decided ``1`` there (0 for frozen positions), so a decoder's CRC verdict
  is ``xor of columns over set bits == crc_offset``;
* ``encoder_columns``: per payload bit, its contribution to the CRC remainder
  the encoder appends.

Both come from the same linear-register identity
``reg(b_0..b_{L-1}) = Z^L(init) xor  XOR_j b_j Z^{L-1-j}(poly)`` where ``Z``
clocks one zero bit; see :func:`_register_columns`.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass
from pathlib import Path

import numpy as np

__all__ = [
    "CRC_POLYS",
    "CrcSpec",
    "CodeConfig",
    "polar_transform",
    "bhattacharyya_profile",
    "construct_frozen_mask",
    "crc_compute",
    "crc_check",
    "crc_check_rows",
    "insert_message",
    "extract_message",
    "load_frozen_mask",
    "save_frozen_mask",
]

# Generator polynomials without the implicit leading term (reference polar.py:37-41).
CRC_POLYS = {8: 0x07, 16: 0x1021, 24: 0x864CFB}


def _log2_exact(N: int) -> int:
    N = int(N)
    if N < 1 or N & (N - 1):
        raise ValueError(f"block length must be a positive power of two, got {N}")
    return N.bit_length() - 1


@dataclass(frozen=True)
class CrcSpec:
    """Register width, generator (low ``width`` coefficients) and seed."""

    width: int
    poly: int
    init: int = 0

    def __post_init__(self):
        if self.width not in CRC_POLYS:
            raise ValueError(f"unsupported CRC width {self.width}, expected 8, 16 or 24")
        top = 1 << self.width
        if not 0 < self.poly < top:
            raise ValueError("CRC polynomial out of range for the given width")
        if not 0 <= self.init < top:
            raise ValueError("CRC initial value out of range for the given width")

    @classmethod
    def standard(cls, width: int) -> "CrcSpec":
        if width not in CRC_POLYS:
            raise ValueError(f"no default polynomial for CRC width {width}")
        return cls(width=width, poly=CRC_POLYS[width])

    @property
    def mask(self) -> int:
        return (1 << self.width) - 1

    def clock_zero(self, reg: int) -> int:
        """One register step with an input bit of 0."""
        top = (reg >> (self.width - 1)) & 1
        reg = (reg << 1) & self.mask
        return reg ^ self.poly if top else reg


def _run_register(bits, spec: CrcSpec) -> int:
    """MSB-first CRC register over a bit sequence (reference polar.py:147-158)."""
    reg = spec.init
    hi = spec.width - 1
    for b in np.asarray(bits, dtype=np.uint8).tolist():
        fb = (reg >> hi) & 1
        reg = (reg << 1) & spec.mask
        if fb != b:
            reg ^= spec.poly
    return reg


def _reg_to_bits(reg: int, width: int) -> np.ndarray:
    return ((reg >> np.arange(width - 1, -1, -1)) & 1).astype(np.uint8)


@functools.lru_cache(maxsize=None)
def _register_columns(length: int, spec: CrcSpec):
    """Affine form of the register over ``length`` input bits.

    Returns ``(cols, offset)``: ``cols[j]`` is the register change caused by a
    1 at input ``j``; ``offset`` is the register after ``length`` zero bits.
    Built backwards in O(length): the last bit contributes ``poly`` and every
    earlier bit contributes one more zero-clock of it.
    """
    cols = np.zeros(length, dtype=np.uint32)
    c = spec.poly
    for j in range(length - 1, -1, -1):
        cols[j] = c
        c = spec.clock_zero(c)
    off = spec.init
    for _ in range(length):
        off = spec.clock_zero(off)
    cols.setflags(write=False)
    return cols, int(off)


def polar_transform(u: np.ndarray) -> np.ndarray:
    """x = u F^{(x)n} in natural order (reference polar.py:79-103).

    Stage ``h`` (1, 2, 4, ...) XORs position ``b*2h + h + t`` into
    ``b*2h + t``; the map is an involution.  Accepts a batch ``[..., N]``.
    """
    u = np.asarray(u)
    N = u.shape[-1] if u.ndim else 0
    _log2_exact(N)
    x = np.array(u, dtype=np.uint8, copy=True)
    lead = x.shape[:-1]
    h = 1
    while h < N:
        v = x.reshape(*lead, N // (2 * h), 2, h)
        v[..., 0, :] ^= v[..., 1, :]
        h <<= 1
    return x


def bhattacharyya_profile(N: int, design_param: float = 0.5) -> np.ndarray:
    """BEC erasure bounds; parent z yields (2z - z^2, z^2) (reference polar.py:106-123)."""
    if not 0.0 < design_param < 1.0:
        raise ValueError(f"design parameter must lie in (0, 1), got {design_param}")
    n = _log2_exact(N)
    z = np.full(1, design_param, dtype=np.float64)
    for _ in range(n):
        worse = 2.0 * z - z * z
        better = z * z
        z = np.stack([worse, better], axis=1).reshape(-1)
    return z


def construct_frozen_mask(N: int, k: int, design_param: float = 0.5) -> np.ndarray:
    """Freeze the N-k largest-z positions, lower index first on ties (polar.py:126-144)."""
    if not 0 < k <= N:
        raise ValueError(f"need 0 < k <= N, got k={k}, N={N}")
    z = bhattacharyya_profile(N, design_param)
    rank = np.argsort(-z, kind="stable")
    mask = np.zeros(N, dtype=np.uint8)
    mask[rank[: N - k]] = 1
    return mask


def crc_compute(message: np.ndarray, spec: CrcSpec) -> np.ndarray:
    """Remainder bits, MSB first, that make ``message || crc`` check clean."""
    return _reg_to_bits(_run_register(message, spec), spec.width)


def crc_check(data: np.ndarray, spec: CrcSpec) -> bool:
    data = np.asarray(data)
    if data.size < spec.width:
        raise ValueError("data shorter than the CRC itself")
    return _run_register(data, spec) == 0


def crc_check_rows(data_rows: np.ndarray, spec: CrcSpec) -> np.ndarray:
    """Row-wise :func:`crc_check` through the affine column table."""
    rows = np.atleast_2d(np.asarray(data_rows, dtype=np.uint8))
    if rows.shape[1] < spec.width:
        raise ValueError("data shorter than the CRC itself")
    cols, off = _register_columns(rows.shape[1], spec)
    syn = np.bitwise_xor.reduce(np.where(rows.astype(bool), cols[None, :], 0), axis=1)
    return (syn.astype(np.uint64) ^ off) == 0


class CodeConfig:
    """Block length N, non-frozen count k (payload + CRC), frozen mask, CRC.

    Mirrors reference ``polar.py:216-286`` (same validation messages).
    """

    def __init__(self, N, k, frozen_mask=None, crc=None, design_param=0.5):
        self.n = _log2_exact(N)
        self.N = int(N)
        self.k = int(k)
        if not 0 < self.k <= self.N:
            raise ValueError(f"need 0 < k <= N, got k={k}, N={N}")
        if isinstance(crc, int) and not isinstance(crc, bool):
            crc = CrcSpec.standard(crc)
        self.crc = crc
        if crc is not None and crc.width >= self.k:
            raise ValueError(f"CRC width {crc.width} does not leave room for message bits (k={k})")
        self.design_param = float(design_param)
        self.bhattacharyya = bhattacharyya_profile(self.N, self.design_param)
        if frozen_mask is None:
            frozen_mask = construct_frozen_mask(self.N, self.k, self.design_param)
        mask = np.asarray(frozen_mask, dtype=np.uint8)
        if mask.shape != (self.N,):
            raise ValueError(f"frozen mask must have length N={N}")
        if np.any(mask > 1):
            raise ValueError("frozen mask entries must be 0 or 1")
        if int(mask.sum()) != self.N - self.k:
            raise ValueError(
                f"frozen mask freezes {int(mask.sum())} positions, expected N-k={self.N - self.k}"
            )
        self.frozen_mask = mask
        self.info_positions = np.flatnonzero(mask == 0)

    @property
    def crc_width(self) -> int:
        return 0 if self.crc is None else self.crc.width

    @property
    def message_len(self) -> int:
        return self.k - self.crc_width

    @property
    def rate(self) -> float:
        return self.k / self.N

    @property
    def message_rate(self) -> float:
        return self.message_len / self.N

    # --- device tables -------------------------------------------------

    def crc_columns(self):
        """(cols[N] uint32, offset): decoder CRC verdict as an affine map on u_hat."""
        cols = np.zeros(self.N, dtype=np.uint32)
        if self.crc is None:
            return cols, 0
        c, off = _register_columns(self.k, self.crc)
        cols[self.info_positions] = c
        return cols, off

    def encoder_columns(self):
        """(cols[m] uint32, offset): CRC remainder register as an affine map on the payload."""
        if self.crc is None:
            return np.zeros(self.message_len, dtype=np.uint32), 0
        c, off = _register_columns(self.message_len, self.crc)
        return np.array(c), off

    def __repr__(self):
        tail = "" if self.crc is None else f", crc={self.crc.width}"
        return f"CodeConfig(N={self.N}, k={self.k}{tail})"


def insert_message(message: np.ndarray, cfg: CodeConfig) -> np.ndarray:
    """Encoder input u: payload then CRC at the info positions, zeros elsewhere."""
    message = np.asarray(message, dtype=np.uint8)
    if message.size != cfg.message_len:
        raise ValueError(f"message has {message.size} bits, config expects {cfg.message_len}")
    u = np.zeros(cfg.N, dtype=np.uint8)
    if cfg.crc is None:
        u[cfg.info_positions] = message
    else:
        u[cfg.info_positions] = np.concatenate([message, crc_compute(message, cfg.crc)])
    return u


def extract_message(u_hat: np.ndarray, cfg: CodeConfig) -> np.ndarray:
    """The k non-frozen decisions (payload followed by CRC)."""
    u_hat = np.asarray(u_hat)
    if u_hat.size != cfg.N:
        raise ValueError(f"decision vector has {u_hat.size} bits, expected N={cfg.N}")
    return u_hat[cfg.info_positions].astype(np.uint8)


def save_frozen_mask(mask: np.ndarray, path) -> None:
    bits = np.asarray(mask, dtype=np.uint8)
    Path(path).write_text(bytes((bits + ord("0")).tolist()).decode("ascii") + "\n")


def load_frozen_mask(path) -> np.ndarray:
    text = Path(path).read_text().strip()
    if not text or not set(text) <= {"0", "1"}:
        raise ValueError(f"frozen mask file {path!r} must hold only '0'/'1' characters")
    return (np.frombuffer(text.encode("ascii"), dtype=np.uint8) - ord("0")).astype(np.uint8)
