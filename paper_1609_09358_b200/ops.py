"""The PyTorch extension: the C-ABI (include/polarcuda.h) as torch ops.

``torch.classes.polar.Code`` holds a code's device tables and its sealed
``pc_code_t``; ``torch.ops.polar.bp_decode / scl_decode / hybrid_decode /
gen_frames / encode`` take and return CUDA tensors and launch on the current
stream (csrc/torch_ops.cpp, built in-tree as libpolar_torch_ops.so).  The
helpers below build the ``Code`` from a ``CodeConfig`` and map the reference's
config dataclasses onto the op arguments; results equal the package's batch
APIs bit for bit (tests/test_gpu_ops.py).
"""

from __future__ import annotations

from pathlib import Path

from . import _native as nat

_LIB = Path(__file__).resolve().parent / "libpolar_torch_ops.so"
_LOADED = False
_G_MODES = ("exact", "min")
_STOP_MODES = ("crc", "reencode", "none")


def load():
    """Load the op library once (needs libpolarcuda.so beside it)."""
    global _LOADED
    import torch

    if not _LOADED:
        if not _LIB.exists():
            raise nat.NativeUnavailable(f"{_LIB.name} is not built (run __graft_entry__.build())")
        torch.ops.load_library(str(_LIB))
        _LOADED = True
    return torch.ops.polar


def code(cfg, da_mask=None):
    """torch.classes.polar.Code of a CodeConfig (tables cached per device)."""
    import torch

    load()
    dc = nat.device_code(cfg, da_mask)
    cached = getattr(dc, "_torch_code", None)
    if cached is None:
        s = dc.struct
        cached = torch.classes.polar.Code(cfg.N, cfg.k, cfg.message_len, cfg.crc_width, int(s.crc_offset),
                                          int(s.enc_crc_offset), dc.frozen_bits, dc.crc_cols, dc.info_pos,
                                          dc.enc_cols, dc.da_bits)
        dc._torch_code = cached
    return cached


def bp_decode(llr, cfg, bp_cfg, soft: bool = False):
    """(u_bits, payload_words, iterations, converged, soft_u, soft_x) of bp_decode over a batch."""
    ops = load()
    return ops.bp_decode(code(cfg), llr, bp_cfg.i_max, _G_MODES.index(bp_cfg.g_mode),
                         _STOP_MODES.index(bp_cfg.stop_mode), float(bp_cfg.llr_max), soft)


def scl_decode(llr, cfg, scl_cfg):
    """(u_bits, payload_words, metric, crc_ok, selected_by_crc) of scl_decode over a batch."""
    from .scl import decision_aided_mask

    ops = load()
    da = decision_aided_mask(cfg, scl_cfg.da_threshold) if scl_cfg.da_threshold > 0 else None
    return ops.scl_decode(code(cfg, da), llr, scl_cfg.list_size, scl_cfg.metric_mode == "exact",
                          scl_cfg.f_mode == "exact", scl_cfg.selector == "bitonic")


def hybrid_decode(llr, cfg, bp_cfg, scl_cfg):
    """(payload_words, converged, iterations) of the hybrid: BP with the CRC stop,
    then CRC-aided SCL on the failures, on the current stream."""
    from .scl import decision_aided_mask

    ops = load()
    da = decision_aided_mask(cfg, scl_cfg.da_threshold) if scl_cfg.da_threshold > 0 else None
    return ops.hybrid_decode(code(cfg), code(cfg, da), llr, bp_cfg.i_max, float(bp_cfg.llr_max),
                             scl_cfg.list_size, scl_cfg.metric_mode == "exact", scl_cfg.f_mode == "exact")


def gen_frames(cfg, seed: int, point: int, frame0: int, count: int, sigma: float):
    """(message words, LLRs) of keyed synthetic frames."""
    return load().gen_frames(code(cfg), seed, point, frame0, count, float(sigma))
