"""The Monte Carlo driver (sim.run_sweep) on the device decoders against the
reference's own committed simulator outputs (plot-tool fixtures, golden_meta
"fixtures"): same keyed frames, same stopping rule, so the non-timing columns
must reproduce.  BP-only points may differ on near-tie frames (fp32 vs fp64
past ~20 iterations); those rows are held to a small tolerance."""

import pytest

from paper_1609_09358_b200 import SimConfig, run_sweep

pytestmark = pytest.mark.gpu


def _parse(cfgline):
    kw = {}
    for item in cfgline.split():
        k, v = item.split("=", 1)
        if k == "ebno_points":
            kw[k] = tuple(float(x) for x in v.split(":"))
        elif k in ("frozen_file",):
            kw[k] = None if v == "None" else v
        elif v in ("True", "False"):
            kw[k] = v == "True"
        else:
            try:
                kw[k] = int(v)
            except ValueError:
                try:
                    kw[k] = float(v)
                except ValueError:
                    kw[k] = v
    return SimConfig(**kw)


@pytest.mark.parametrize("name", ["hybrid_sweep", "scl_sweep", "no_timing", "bp_sweep"])
def test_sweep_reproduces_reference_fixture(golden_meta, name):
    fx = golden_meta["fixtures"][name]
    cfg = _parse(fx["config"])
    recs = run_sweep(cfg)
    assert len(recs) == len(fx["rows"])
    for rec, row in zip(recs, fx["rows"]):
        assert rec.ebno_db == float(row["ebno_db"])
        if cfg.decoder == "bp":
            # a near-tie BP frame (fp32 vs fp64 past ~20 iterations) that flips its
            # error changes where the min-frame-errors rule stops: the next error
            # can be tens of frames later, so rows are held to the error count and
            # a 10% frame window
            assert abs(rec.frames - int(row["frames"])) <= max(2, int(0.10 * int(row["frames"]))), (rec, row)
            assert abs(rec.frame_errors - int(row["frame_errors"])) <= 1, (rec, row)
            continue
        assert rec.frames == int(row["frames"]), (rec, row)
        assert rec.frame_errors == int(row["frame_errors"]), (rec, row)
        assert rec.bit_errors == int(row["bit_errors"]), (rec, row)
        if row["gamma_bp_fer"]:
            assert abs(rec.gamma_bp_fer - float(row["gamma_bp_fer"])) <= 2.0 / rec.frames, (rec, row)


def test_cli_no_timing_is_byte_identical_to_reference_fixture(golden_meta, tmp_path):
    """The reference's --no-timing CSV (plot-tool fixture no_timing.csv, config
    N=128 k=64 scl L=2, 2 and 3 dB, seed 14) reproduced byte for byte through
    the CLI (reference cli.py:72-115, test_acceptance.py:311-331)."""
    from paper_1609_09358_b200.cli import main

    out = tmp_path / "sweep.csv"
    rc = main(["--n", "128", "--k", "64", "--decoder", "scl", "--list-size", "2", "--ebno", "2:3:1",
               "--seed", "14", "--min-frame-errors", "10", "--max-frames", "500", "--no-timing",
               "--out", str(out)])
    assert rc == 0
    assert out.read_text() == golden_meta["fixtures"]["no_timing"]["raw"]
