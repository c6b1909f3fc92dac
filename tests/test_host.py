"""Host-side contracts on CPU: code construction, CRC tables, channel, API
validation, C-ABI exports, the multi-GPU sharding plan (gloo)."""

import binascii
import ctypes
import math
import re

import numpy as np
import pytest

from conftest import ROOT, unpack
import paper_1609_09358_b200 as ps
from paper_1609_09358_b200 import (
    BpConfig,
    CodeConfig,
    CrcSpec,
    SclConfig,
    SimConfig,
    bitonic_sort_select,
    crc_check,
    crc_check_rows,
    crc_compute,
    g_fn,
    init_graph,
    pe_endpoints,
    pseudo_sort_select,
    stopping_check,
    theoretical_throughput,
)
from paper_1609_09358_b200 import _native as nat
from paper_1609_09358_b200.channel import make_frame


# ------------------------------------------------------------ construction --

def test_frozen_masks_match_reference_golden(golden):
    for key in golden:
        if key.startswith("mask_"):
            _, N, k = key.split("_")
            code = CodeConfig(int(N), int(k))
            assert np.array_equal(code.frozen_mask, unpack(golden[key], int(N))), key


def test_bhattacharyya_small_profiles():
    assert ps.bhattacharyya_profile(1).tolist() == [0.5]
    assert ps.bhattacharyya_profile(2).tolist() == [0.75, 0.25]
    assert ps.bhattacharyya_profile(4).tolist() == [0.9375, 0.5625, 0.4375, 0.0625]
    assert np.flatnonzero(ps.construct_frozen_mask(8, 4)).tolist() == [0, 1, 2, 4]


def test_transform_involution_and_matrix():
    rng = np.random.default_rng(1)
    g = np.array([[1]], np.int64)
    for _ in range(6):
        g = np.kron(g, np.array([[1, 0], [1, 1]]))
    u = rng.integers(0, 2, (100, 64)).astype(np.uint8)
    assert np.array_equal(ps.polar_transform(u), (u.astype(np.int64) @ g) & 1)
    assert np.array_equal(ps.polar_transform(ps.polar_transform(u)), u)


def test_crc_known_answers_and_golden(golden):
    data = np.unpackbits(np.frombuffer(b"123456789", np.uint8))
    v16 = int("".join(map(str, crc_compute(data, CrcSpec.standard(16)))), 2)
    assert v16 == 0x31C3 == binascii.crc_hqx(b"123456789", 0)
    assert int("".join(map(str, crc_compute(data, CrcSpec.standard(8)))), 2) == 0xF4
    for w, m, L, out in zip(golden["crc_widths"], golden["crc_msgs"], golden["crc_lens"], golden["crc_out"]):
        msg = unpack(m, 1008)[:L]
        assert np.array_equal(crc_compute(msg, CrcSpec.standard(int(w))), unpack(out, 24)[:w])


def test_crc_affine_tables_equal_register():
    rng = np.random.default_rng(2)
    for w in (8, 16, 24):
        code = CodeConfig(256, 128, crc=w)
        cols, off = code.crc_columns()
        ecols, eoff = code.encoder_columns()
        for _ in range(20):
            u = rng.integers(0, 2, 256).astype(np.uint8) * (1 - code.frozen_mask)
            syn = np.bitwise_xor.reduce(np.where(u.astype(bool), cols, 0))
            assert (syn == off) == crc_check(u[code.info_positions], code.crc)
            msg = rng.integers(0, 2, code.message_len).astype(np.uint8)
            reg = int(np.bitwise_xor.reduce(np.where(msg.astype(bool), ecols, 0))) ^ eoff
            bits = [(reg >> (w - 1 - b)) & 1 for b in range(w)]
            assert bits == crc_compute(msg, code.crc).tolist()
    rows = rng.integers(0, 2, (30, 128)).astype(np.uint8)
    spec = CrcSpec.standard(16)
    assert np.array_equal(crc_check_rows(rows, spec), [crc_check(r, spec) for r in rows])


def test_host_frame_generator_matches_reference_golden(golden):
    code = CodeConfig(1024, 512, crc=16)
    sigma = ps.ebno_to_sigma(2.0, code.rate)
    for f in range(3):
        m, l = make_frame(code, sigma, ps.frame_rng(99, 1, f))
        assert np.array_equal(m, unpack(golden["gen_msgs"][f], code.message_len))
        assert np.array_equal(l, golden["gen_llrs"][f])


def test_code_config_validation():
    with pytest.raises(ValueError):
        CodeConfig(12, 6)
    with pytest.raises(ValueError):
        CodeConfig(16, 0)
    with pytest.raises(ValueError):
        CodeConfig(16, 8, crc=16)
    with pytest.raises(ValueError):
        CodeConfig(8, 4, frozen_mask=np.ones(8))
    code = CodeConfig(1024, 528, crc=16)
    assert code.rate == 528 / 1024 and code.message_len == 512


def test_frozen_mask_file_roundtrip(tmp_path):
    mask = ps.construct_frozen_mask(64, 20)
    p = tmp_path / "m.txt"
    ps.save_frozen_mask(mask, p)
    assert np.array_equal(ps.load_frozen_mask(p), mask)
    (tmp_path / "bad.txt").write_text("0102\n")
    with pytest.raises(ValueError):
        ps.load_frozen_mask(tmp_path / "bad.txt")


# ---------------------------------------------------------- API utilities --

def test_bp_host_helpers():
    assert float(g_fn(20.0, 20.0)) == pytest.approx(19.306852819440056, abs=1e-12)
    assert pe_endpoints(3, 5) == (9, 13)
    with pytest.raises(ValueError):
        pe_endpoints(0, 0)
    code = CodeConfig(8, 4)
    g = init_graph(np.linspace(-30, 30, 8), code, BpConfig())
    assert np.all(np.abs(g.l_msgs[3]) <= 20) and np.array_equal(g.r_msgs[0], 20.0 * code.frozen_mask)
    with pytest.raises(ValueError):
        stopping_check(init_graph(np.zeros(8), code, BpConfig(stop_mode="crc")), code, BpConfig(stop_mode="crc"))
    with pytest.raises(ValueError):
        BpConfig(i_max=0)
    with pytest.raises(ValueError):
        SclConfig(selector="quick")


def test_selectors_match_full_sort():
    rng = np.random.default_rng(8)
    for L in (1, 2, 4, 8, 16, 32):
        for _ in range(100):
            m = rng.normal(0, 3, 2 * L)
            if rng.random() < 0.5:
                m = np.round(m)
            m[rng.random(m.size) < 0.2] = np.inf
            order = np.lexsort((np.arange(m.size), m))
            ref = order[np.isfinite(m[order])][:L]
            assert np.array_equal(pseudo_sort_select(m, L), ref)
            assert np.array_equal(bitonic_sort_select(m, L), ref)


def test_scalar_helpers_known_answers():
    assert ps.sc_f(1.0, 1.0, exact=True) == pytest.approx(0.4337808304830273, abs=1e-15)
    assert ps.sc_f(-3.0, 5.0) == -3.0 and ps.sc_f(0.0, 4.0) == 0.0
    assert ps.sc_g(2.0, 5.0, 1) == 3.0
    assert ps.path_metric_update(0.0, 30.0, 0) == pytest.approx(9.357622968839737e-14)
    assert ps.path_metric_update(0.0, 0.0, 1) == pytest.approx(math.log(2))


def test_throughput_model():
    assert theoretical_throughput(100.0, 1.0, 0.01) == pytest.approx(50.0)
    assert theoretical_throughput(10.0, 10.0, 1.0) == pytest.approx(5.0)
    with pytest.raises(ValueError):
        theoretical_throughput(1.0, 1.0, 1.5)


def test_sim_config_validation():
    with pytest.raises(ValueError):
        SimConfig(N=64, k=32, decoder="magic", ebno_points=(1.0,))
    with pytest.raises(ValueError):
        SimConfig(N=64, k=32)
    assert ps.CSV_HEADER.split(",")[0] == "ebno_db" and len(ps.CSV_HEADER.split(",")) == 12


# --------------------------------------------------------------- the C-ABI --

def test_c_abi_library_exports_every_declared_symbol():
    lib = nat.load()
    header = (ROOT / "include" / "polarcuda.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(pc_\w+)\(", header, re.M))
    assert declared == set(nat.EXPORTS)
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.pc_version() == 1
    assert lib.pc_strerror(-1) == b"invalid argument"
    assert lib.pc_workspace_bytes() >= 4


def test_c_abi_rejects_bad_arguments_without_gpu():
    lib = nat.load()
    bad = nat.PcCode(12, 3, 6, 6, 0, 0, 0, 0, None, None, None, None, None)
    cfg = nat.PcBpCfg(50, 0, 0, 0, 20.0)
    assert lib.pc_bp_decode(None, 1, ctypes.byref(bad), ctypes.byref(cfg), None, None, None, None, None, None,
                            None, None) == -1
    assert lib.pc_compact(None, -1, None, None, None, None) == -1


def test_decoders_fail_loudly_without_device():
    if nat.load().pc_device_count() > 0:
        pytest.skip("a device is present")
    code = CodeConfig(64, 32, crc=8)
    with pytest.raises(nat.NativeUnavailable):
        ps.bp_decode(np.zeros(64), code, BpConfig(stop_mode="crc"))
    with pytest.raises(nat.NativeUnavailable):
        ps.scl_decode(np.zeros(64), code)


def test_product_path_does_not_import_the_oracle():
    pkg = ROOT / "paper_1609_09358_b200"
    for p in pkg.rglob("*.py"):
        assert not re.search(r"^\s*(from|import)\s+oracle", p.read_text(), re.M), p


def test_cli_parser_matches_reference_flags():
    from paper_1609_09358_b200.cli import _parse_ebno_range, build_parser, config_from_args

    assert _parse_ebno_range("1:4:0.5") == (1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0)
    assert _parse_ebno_range("2:3:1") == (2.0, 3.0)
    args = build_parser().parse_args(["--n", "1024", "--rate", "0.5", "--decoder", "hybrid", "--list-size", "32",
                                      "--ebno-list", "1,2.5", "--crc", "none", "--no-timing"])
    cfg = config_from_args(args)
    assert (cfg.N, cfg.k, cfg.decoder, cfg.list_size, cfg.crc_width) == (1024, 512, "hybrid", 32, 0)
    assert cfg.ebno_points == (1.0, 2.5) and cfg.measure_time is False
    with pytest.raises(SystemExit):
        build_parser().parse_args(["--n", "8", "--k", "4", "--rate", "0.5", "--ebno", "1:2:1"])


def test_scl_workspace_size_query_without_gpu():
    """pc_scl_workspace_bytes sizes the K3 traceback from the code (no device
    needed: it falls back to 148 SMs); bad configurations return -1."""
    lib = nat.load()

    def code_struct(N, k, crc=16):
        return nat.PcCode(N, int(np.log2(N)), k, k - crc, crc, 0, 0, N - k, 1, 1, 1, 1, None)

    small = lib.pc_scl_workspace_bytes(ctypes.byref(code_struct(1024, 512)), ctypes.byref(ps.SclConfig(32).native()))
    large = lib.pc_scl_workspace_bytes(ctypes.byref(code_struct(4096, 2048)), ctypes.byref(ps.SclConfig(32).native()))
    assert small > 256 and large > 256  # resident warps x windows x 160 B
    bad = ps.SclConfig(32).native()
    bad.L = 33  # list sizes 1..32 (any; N >= 64 when not a power of two)
    assert lib.pc_scl_workspace_bytes(ctypes.byref(code_struct(1024, 512)), ctypes.byref(bad)) == -1
    # v2 (N < 32) needs only the counter block
    assert lib.pc_scl_workspace_bytes(ctypes.byref(code_struct(16, 8, 0)), ctypes.byref(ps.SclConfig(4).native())) \
        == lib.pc_workspace_bytes()


def test_c_abi_refuses_unsealed_code_without_gpu():
    """A code struct that pc_code_seal never validated (or that changed after
    sealing) is refused before any launch: first_info is derived by the
    library, never trusted from the caller."""
    lib = nat.load()
    code = nat.PcCode(1024, 10, 512, 496, 16, 0, 0, 191, 16, 16, 16, 16, None)
    cfg = nat.PcBpCfg(50, 0, 0, 0, 20.0)
    assert lib.pc_bp_decode(16, 1, ctypes.byref(code), ctypes.byref(cfg), None, None, None, None, 16, 16,
                            None, None) == -1
    scfg = ps.SclConfig(32).native()
    assert lib.pc_scl_decode(16, 1, None, None, ctypes.byref(code), ctypes.byref(scfg), None, None, None, None,
                             None, None, 16, None) == -1
    assert lib.pc_encode(16, 1, ctypes.byref(code), 16, None) == -1


def test_stage_busy_time_is_the_union_of_intervals():
    """hybrid._busy: a stage's service time with concurrent chunks (several SCL
    streams) is the measure of the union of their [start, end) intervals."""
    from paper_1609_09358_b200.hybrid import _busy

    assert _busy([], []) == 0.0
    assert _busy([0], [10]) == pytest.approx(10e-9)
    assert _busy([0, 5, 20], [10, 12, 25]) == pytest.approx(17e-9)  # overlap merged
    assert _busy([20, 0], [30, 10]) == pytest.approx(20e-9)  # disjoint: the sum
    big = 1_760_000_000_000_000_000  # globaltimer-sized int64 stamps keep ns resolution
    assert _busy([big, big + 3], [big + 5, big + 7]) == pytest.approx(7e-9)
