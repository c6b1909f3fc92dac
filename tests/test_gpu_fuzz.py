"""A fixed slice of the randomized device-vs-oracle sweep (tests/parity/fuzz_parity.py):
random codes N = 2..4096 (any rate, CRC none/8/16/24), channel points, batch
sizes and every decoder knob.  SCL must equal the oracle on every frame
(except fp64-rounding-limited exact-f frames, certified per frame); BP may
part only on the near-tie class (a small fraction)."""
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, str(Path(__file__).resolve().parent / "parity"))


@pytest.mark.parametrize("seed", [11, 12])
def test_random_configurations_match_the_oracle(seed):
    import fuzz_parity

    fails, scl_bad, bp_diff, bp_frames = fuzz_parity.run(80, seed, verbose=False)
    assert not fails, fails
    assert bp_diff <= max(3, 0.02 * bp_frames), (bp_diff, bp_frames)
