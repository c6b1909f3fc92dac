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

# ---- the reference's own test suite (tests/ref_suite) ----
# tests/ref_suite/vendor.py copies /root/reference/pkg/tests/*.py, unmodified,
# into the git-ignored tests/ref_suite/vendor/; they import ``polarsim``, the
# test-only alias of this package in tests/ref_suite/polarsim/.  Every vendored
# test is marked ``gpu`` (the decoders run on the device; on a CPU host they
# raise NativeUnavailable by design) and ``ref_suite``.  Failures that follow
# from the documented fp32 device arithmetic are strict xfails, with the cause
# here and in DESIGN.md section 4.
REF_SUITE = Path(__file__).resolve().parent / "ref_suite"
if str(REF_SUITE) not in sys.path:
    sys.path.insert(0, str(REF_SUITE))
# the reference's CLI test runs `python -m polarsim` in a subprocess
os.environ["PYTHONPATH"] = os.pathsep.join([str(REF_SUITE), str(ROOT)] +
                                           [p for p in [os.environ.get("PYTHONPATH")] if p])
_FP32 = ("fp64 exact-equality assertion on device fp32 arithmetic (north_star: BP/SCL messages within 1e-4 "
         "relative in fp32); measured on the B200: ")
REF_XFAIL: dict[str, str] = {
    # test_bp.py:126-141: assert_array_equal of iterate_once messages against the
    # scalar fp64 restatement (reference_impls.py:154-188)
    "test_bp.py::test_iteration_matches_scalar_reference": _FP32 + "max |diff| 4.5e-7, max relative 1.2e-7",
    # test_bp.py:144-152: hand trace at abs=1e-15
    "test_bp.py::test_first_sweep_hand_trace_n2": _FP32 + "4.99999952 vs 4.99999969 (|diff| 1.7e-7)",
    # test_scl.py:200-214: metric against a brute-force fp64 forced-path metric at
    # abs=1e-12; the WINNER (the minimum-metric codeword) is the same, only the
    # fp32 metric value differs (8e-8)
    "test_scl.py::test_metric_minimal_among_all_messages": _FP32 + "4.99495935 vs 4.99495944 (|diff| 8.2e-8)",
}


def pytest_collection_modifyitems(config, items):
    vend = REF_SUITE / "vendor"
    for it in items:
        path = Path(str(it.fspath))
        if vend not in path.parents:
            continue
        it.add_marker(pytest.mark.gpu)
        it.add_marker(pytest.mark.ref_suite)
        key = f"{path.name}::{it.name}"
        if key in REF_XFAIL:
            it.add_marker(pytest.mark.xfail(reason=REF_XFAIL[key], strict=True))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libpolarcuda.so")
    config.addinivalue_line("markers", "slow: long-running statistical check")
    config.addinivalue_line("markers", "ref_suite: the reference's own tests (tests/ref_suite) on this package")


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
    # (its own numba cache: entries written under the module name "polarsim" do not load as "polarsim_ref")
    os.environ["NUMBA_CACHE_DIR"] = "/tmp/numba_cache_polarsim_ref"
    # loaded under its own name: "polarsim" is the test-only alias of this
    # package that the vendored reference suite imports (tests/ref_suite)
    if "polarsim_ref" not in sys.modules:
        import importlib.util

        spec = importlib.util.spec_from_file_location("polarsim_ref", REF_SRC / "polarsim" / "__init__.py",
                                                      submodule_search_locations=[str(REF_SRC / "polarsim")])
        mod = importlib.util.module_from_spec(spec)
        sys.modules["polarsim_ref"] = mod
        spec.loader.exec_module(mod)
    return sys.modules["polarsim_ref"]


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
