"""Shared fixtures.  `-m gpu` tests need a B200 and the built libpolarcuda.so;
everything else runs on CPU.  /root/reference is used only when present (dev
container); the GPU box sees the committed golden fixtures instead."""

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"
REF_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libpolarcuda.so")
    config.addinivalue_line("markers", "slow: long-running statistical check")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN / "golden.npz"))


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden_meta.json").read_text())


@pytest.fixture(scope="session")
def reference():
    """The live reference package, only where /root/reference exists."""
    if not REF_SRC.exists():
        pytest.skip("reference tree not present (GPU box); golden fixtures cover it")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_tests")
    if str(REF_SRC) not in sys.path:
        sys.path.append(str(REF_SRC))
    import polarsim

    return polarsim


def unpack(packed, L):
    return np.unpackbits(np.asarray(packed, np.uint8), axis=-1, bitorder="little")[..., :L]


def golden_frames(meta_set, code):
    """Regenerate a golden set's frames with the host generator (fp32-rounded LLRs)."""
    from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame

    sigma = ebno_to_sigma(meta_set["ebno"], code.rate)
    msgs, llrs = [], []
    for f in range(meta_set["count"]):
        m, l = make_frame(code, sigma, frame_rng(meta_set["seed"], meta_set["point"], f))
        msgs.append(m)
        llrs.append(l.astype(np.float32).astype(np.float64))
    return np.array(msgs), np.array(llrs)


def gpu_available():
    try:
        from paper_1609_09358_b200 import _native as nat
        import torch

        return torch.cuda.is_available() and nat.load().pc_device_count() > 0
    except Exception:
        return False
