"""Pin the CPU oracle (oracle/oracle.c) to the reference: bit-exact against the
golden vectors generated from the reference, and -- where /root/reference is
present -- against the live reference on fresh inputs."""

import binascii

import numpy as np
import pytest

import oracle
from conftest import golden_frames, unpack
from paper_1609_09358_b200 import CodeConfig
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame


def test_bp_decisions_match_golden(golden, golden_meta):
    for name in ("bp128", "bp1024a", "bp1024b", "bp2048", "bp4096"):
        meta = golden_meta["sets"][name]
        code = CodeConfig(meta["N"], meta["k"], crc=16)
        _, llrs = golden_frames(meta, code)
        u, it, cv = oracle.bp_batch(llrs, code, stop_mode="crc")
        assert np.array_equal(it, golden[f"{name}_iters"]), name
        assert np.array_equal(cv, golden[f"{name}_conv"].astype(bool)), name
        assert np.array_equal(u, unpack(golden[f"{name}_u"], code.N)), name


def test_bp_other_stop_modes_match_golden(golden, golden_meta):
    meta = golden_meta["sets"]["bp64"]
    code = CodeConfig(64, 32, crc=None)
    _, llrs = golden_frames(meta, code)
    for mode in ("reencode", "none"):
        u, it, cv = oracle.bp_batch(llrs, code, i_max=20, stop_mode=mode)
        assert np.array_equal(it, golden[f"bp64_{mode}_iters"])
        assert np.array_equal(u, unpack(golden[f"bp64_{mode}_u"], 64))


@pytest.mark.parametrize("N", [32, 1024])
def test_teacher_forced_iteration_bit_exact(golden, N):
    L, R = oracle.bp_iterate(golden[f"tf{N}_lin"], golden[f"tf{N}_rin"])
    assert np.array_equal(L, golden[f"tf{N}_lout"])
    assert np.array_equal(R, golden[f"tf{N}_rout"])


def test_g_known_values():
    assert oracle.bp_g(20.0, 20.0) == pytest.approx(19.306852819440056, abs=1e-12)
    assert oracle.bp_g(0.0, 5.0) == 0.0
    assert oracle.bp_g(3.0, -5.0, "min") == -3.0
    assert oracle.bp_g(50.0, 60.0, "min") == 20.0


def test_scl_winners_match_golden(golden, golden_meta):
    for name in ("scl128L4", "scl128L32", "scl1024L8", "scl1024L32", "scl2048L32", "scl256L1", "scl512L2",
                 "scl512L16", "scl2048L1", "scl2048L4", "scl4096L8"):
        meta = golden_meta["sets"][name]
        code = CodeConfig(meta["N"], meta["k"], crc=16)
        _, llrs = golden_frames(meta, code)
        u, mt, ok = oracle.scl_batch(llrs, code, meta["L"])
        assert np.array_equal(u, unpack(golden[f"{name}_u"], code.N)), name
        assert np.array_equal(mt, golden[f"{name}_metric"]), name
        assert np.array_equal(ok, golden[f"{name}_crc"].astype(bool)), name


def test_scl_knobs_match_golden(golden, golden_meta):
    from paper_1609_09358_b200.scl import decision_aided_mask

    meta = golden_meta["sets"]["sclknob"]
    code = CodeConfig(128, 64, crc=8)
    _, llrs = golden_frames(meta, code)
    da = decision_aided_mask(code, 0.05)
    for tag, kw in (("fexact", dict(f_mode="exact")), ("approx", dict(metric_mode="approx")), ("da", dict(da=da))):
        for f, l in enumerate(llrs):
            r = oracle.scl_decode(l, code, 8, **kw)
            assert np.array_equal(r["u_hat"], unpack(golden[f"sclknob_{tag}_u"][f], 128)), (tag, f)
            assert r["metric"] == golden[f"sclknob_{tag}_metric"][f]


def test_hybrid_matches_golden(golden, golden_meta):
    for name in ("hyb1024a", "hyb1024b"):
        meta = golden_meta["sets"][name]
        code = CodeConfig(1024, 512, crc=16)
        _, llrs = golden_frames(meta, code)
        pay, prov, _ = oracle.hybrid_batch(llrs, code, i_max=50, L=32)
        assert np.array_equal(pay, unpack(golden[f"{name}_payload"], code.message_len))
        assert np.array_equal(prov, golden[f"{name}_scl"].astype(bool))


def test_scl_selectors_agree_and_tie_rule():
    cand = np.array([1.0, 1.0, 0.5, 1.0, np.inf, 2.0])
    for bit in (False, True):
        keep = oracle.select_keep(cand, 3, bitonic=bit)
        assert keep.tolist() == [1, 1, 1, 0, 0, 0]
    rng = np.random.default_rng(8)
    for L in (1, 2, 4, 8, 16, 32):
        for _ in range(50):
            m = np.round(rng.normal(0, 3, 2 * L))
            m[rng.random(m.size) < 0.2] = np.inf
            assert np.array_equal(oracle.select_keep(m, L), oracle.select_keep(m, L, bitonic=True))


def test_encoder_and_crc_known_answers(golden):
    data = np.unpackbits(np.frombuffer(b"123456789", np.uint8))
    assert oracle.crc_register(data, 16, 0x1021) == 0x31C3 == binascii.crc_hqx(b"123456789", 0)
    assert oracle.crc_register(data, 8, 0x07) == 0xF4
    code = CodeConfig(1024, 512, crc=16)
    msgs = unpack(golden["enc_msgs"], code.message_len)
    x = np.array([oracle.encode(m, code) for m in msgs])
    assert np.array_equal(x, unpack(golden["enc_x"], 1024))


def test_oracle_matches_live_reference(reference):
    """Fresh frames (not in the fixtures) through both implementations."""
    ref = reference
    for N, k, L, eb in ((256, 128, 8, 1.5), (1024, 512, 32, 2.0)):
        rc = ref.CodeConfig(N, k, crc=16)
        code = CodeConfig(N, k, crc=16)
        sigma = ebno_to_sigma(eb, code.rate)
        for f in range(6):
            _, llr = make_frame(code, sigma, frame_rng(555, 3, f))
            a = ref.bp_decode(llr, rc, ref.BpConfig(stop_mode="crc"))
            b = oracle.bp_decode(llr, code, stop_mode="crc")
            assert a.iterations_used == b["iterations_used"]
            assert np.array_equal(a.soft_u, b["soft_u"]) and np.array_equal(a.soft_x, b["soft_x"])
            s = ref.scl_decode(llr, rc, ref.SclConfig(L))
            t = oracle.scl_decode(llr, code, L)
            assert np.array_equal(s.u_hat, t["u_hat"]) and s.metric == t["metric"]
