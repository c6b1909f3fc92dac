"""bench.py's JSON-line contract, on tiny workloads: every workload prints one
line with the keys the driver and the judge read."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "cpu_baseline"}


def _line(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [s for s in out.stdout.splitlines() if s.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _line("--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-frames", "4")
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"


@pytest.mark.gpu
@pytest.mark.parametrize("wl,frames", [("c3", 2048), ("c1", 8192), ("c2", 512), ("c4", 256), ("c5", 256)])
def test_workload_lines(wl, frames):
    d = _line("--workload", wl, "--steps", "1", "--warmup", "3", "--frames", str(frames), "--cpu-frames", "8")
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["clocks"]["sm_mhz"] is not None
    assert d["gpu_launches"] >= 1
    if wl in ("c1", "c3", "c4"):
        r = d["roofline"]
        assert r["bound"] in ("issue", "xu") and r["achieved"] > 0 and r["frac_alg"] > 0
        assert 0 < r["frac"] < 1.05 and 0 < r["xu"]["frac"] < 1.0
        assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    if wl == "c1":
        assert d["fixed_cap"]["stop_mode"] == "none" and d["fixed_cap"]["frac_alg"] > 0
    if wl == "c3":
        assert d["k3"]["mframes_per_s"] > 0 and 0 < d["k3"]["share_of_step"] < 1
        ps = d["parity_sample"]  # the cpu_baseline frames through the device: 7 points x 8 frames
        assert ps["frames"] == 56 and ps["payload_identical"] >= 54
        assert d["overlapped"]["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("wl,frames", [("c4", 256), ("c3", 1024)])
def test_gpus_flag_spawns_ranks_and_merges_counters(wl, frames):
    """`bench.py --gpus 2` (no launcher) runs two ranks itself; on the one-GPU
    box both share cuda:0 and merge over gloo.  The merged per-point counters
    equal one rank decoding the same global frames (frames are keyed by their
    global index, shard.shard_range)."""
    common = ("--workload", wl, "--steps", "1", "--warmup", "3", "--no-cpu")
    two = _line("--gpus", "2", "--frames", str(frames), *common)
    one = _line("--frames", str(2 * frames), *common)
    assert two["n_gpus"] == 2 and two["config"]["parallelism"] == "frame-sharded x2"
    assert one["n_gpus"] == 1
    keys = ("frames", "frame_errors", "bit_errors", "bp_iterations")
    for a, b in zip(two["sweep"], one["sweep"]):
        assert {k: a[k] for k in keys} == {k: b[k] for k in keys}
