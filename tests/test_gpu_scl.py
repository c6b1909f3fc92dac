"""K3 (pc_scl_decode) parity: winners bit-identical with the reference on
identical fp32-rounded inputs (golden fixtures) and with the C oracle at
larger scale.  Metrics are fp32 on the device: relative tolerance 1e-4."""

import numpy as np
import pytest

import oracle
from conftest import golden_frames, unpack
from paper_1609_09358_b200 import CodeConfig, SclConfig, scl_decode, scl_decode_batch
from paper_1609_09358_b200.channel import channel_llr, ebno_to_sigma, frame_rng, make_frame, modulate_bpsk
from paper_1609_09358_b200.codes import crc_check, extract_message, insert_message, polar_transform

pytestmark = pytest.mark.gpu

METRIC_RTOL = 1e-4


def _compare(name, ref_u, ref_metric, ref_crc, got, allow=0):
    bad = [f for f in range(len(ref_metric)) if not np.array_equal(got.u_hat[f], ref_u[f])]
    assert len(bad) <= allow, f"{name}: winner differs on frames {bad}"
    good = [f for f in range(len(ref_metric)) if f not in bad]
    assert np.array_equal(got.crc_ok[good], np.asarray(ref_crc, bool)[good])
    np.testing.assert_allclose(got.metric[good], np.asarray(ref_metric)[good], rtol=METRIC_RTOL, atol=1e-5)
    return bad


@pytest.mark.parametrize(
    "name", ["scl128L4", "scl128L32", "scl1024L8", "scl1024L32", "scl2048L32", "scl256L1", "scl512L2", "scl512L16",
             "scl2048L1", "scl2048L4", "scl4096L8"]
)
def test_winners_match_reference(golden, golden_meta, name):
    meta = golden_meta["sets"][name]
    code = CodeConfig(meta["N"], meta["k"], crc=16)
    _, llrs = golden_frames(meta, code)
    got = scl_decode_batch(llrs, code, SclConfig(list_size=meta["L"]))
    _compare(name, unpack(golden[f"{name}_u"], code.N), golden[f"{name}_metric"], golden[f"{name}_crc"], got)


@pytest.mark.parametrize(
    "tag,cfg",
    [("fexact", SclConfig(8, f_mode="exact")), ("approx", SclConfig(8, metric_mode="approx")),
     ("da", SclConfig(8, da_threshold=0.05))],
)
def test_decoder_knobs_match_reference(golden, golden_meta, tag, cfg):
    meta = golden_meta["sets"]["sclknob"]
    code = CodeConfig(128, 64, crc=8)
    _, llrs = golden_frames(meta, code)
    got = scl_decode_batch(llrs, code, cfg)
    ref_u = unpack(golden[f"sclknob_{tag}_u"], 128)
    bad = [f for f in range(len(llrs)) if not np.array_equal(got.u_hat[f], ref_u[f])]
    assert not bad, f"{tag}: {bad}"
    np.testing.assert_allclose(got.metric, golden[f"sclknob_{tag}_metric"], rtol=1e-3, atol=1e-4)


@pytest.mark.parametrize("nv", [0, 1, 2, 3])
def test_virtual_levels_do_not_change_results(nv):
    from paper_1609_09358_b200 import _native as nat
    import ctypes
    import torch

    code = CodeConfig(1024, 512, crc=16)
    sigma = ebno_to_sigma(1.5, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(61, 0, f))[1] for f in range(48)])
    x = torch.from_numpy(llrs.astype(np.float32)).cuda()
    base = scl_decode_batch(x, code, SclConfig(32))
    for wpc in (1, 2, 4):
        cfg = SclConfig(32).native(virtual_levels=nv, warps_per_cta=wpc)
        dc = nat.device_code(code)
        u = torch.zeros_like(base.u_hat)
        mt = torch.zeros_like(base.metric)
        nat.check(nat.load().pc_scl_decode(x.data_ptr(), 48, None, None, dc.ref, ctypes.byref(cfg), u.data_ptr(),
                                           None, mt.data_ptr(), None, None, None, dc.scl_workspace(cfg).data_ptr(),
                                           nat.stream_handle()), "scl")
        assert torch.equal(u, base.u_hat)
        assert torch.equal(mt, base.metric)


@pytest.mark.parametrize("N,L", [(1024, 4), (2048, 8), (2048, 32), (4096, 32)])
def test_compiled_in_kernels_match_runtime_kernels(N, L):
    """The default configuration runs K3 kernels with the code geometry and
    the default knobs compiled in (k_scl3<L, false, 3, n>); two virtual levels
    select the runtime-parameter kernel, which must give the same bits
    (virtual levels never change results)."""
    from paper_1609_09358_b200 import _native as nat
    import ctypes
    import torch

    code = CodeConfig(N, N // 2, crc=16)
    sigma = ebno_to_sigma(1.5, code.rate)
    B = 64
    llrs = np.array([make_frame(code, sigma, frame_rng(62, N, f))[1] for f in range(B)])
    x = torch.from_numpy(llrs.astype(np.float32)).cuda()
    base = scl_decode_batch(x, code, SclConfig(L))
    cfg = SclConfig(L).native(virtual_levels=2)
    dc = nat.device_code(code)
    u = torch.zeros_like(base.u_hat)
    mt = torch.zeros_like(base.metric)
    nat.check(nat.load().pc_scl_decode(x.data_ptr(), B, None, None, dc.ref, ctypes.byref(cfg), u.data_ptr(), None,
                                       mt.data_ptr(), None, None, None, dc.scl_workspace(cfg).data_ptr(),
                                       nat.stream_handle()), "scl")
    assert torch.equal(u, base.u_hat)
    assert torch.equal(mt, base.metric)


@pytest.mark.parametrize("N,k,L,eb,count", [(1024, 512, 32, 1.5, 400), (1024, 512, 4, 1.0, 400),
                                            (2048, 1024, 16, 2.0, 100), (64, 32, 2, 1.0, 400),
                                            (2048, 1024, 32, 1.5, 300), (2048, 1024, 1, 2.0, 1000),
                                            (4096, 2048, 32, 1.5, 48)])
def test_winners_vs_oracle_at_scale(N, k, L, eb, count):
    code = CodeConfig(N, k, crc=16)
    sigma = ebno_to_sigma(eb, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(707, L, f))[1] for f in range(count)])
    llrs = llrs.astype(np.float32).astype(np.float64)
    ref_u, ref_m, ref_ok = oracle.scl_batch(llrs, code, L)
    got = scl_decode_batch(llrs, code, SclConfig(L))

    class Ref:
        pass

    bad = _compare(f"N{N}L{L}", ref_u, ref_m, ref_ok, got, allow=max(0, count // 400))
    print(f"N={N} L={L}: {len(bad)} near-tie frames {bad}")


def test_list_size_one_equals_sc():
    code = CodeConfig(128, 64, crc=None)
    sigma = ebno_to_sigma(1.0, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(128001, 0, f))[1] for f in range(2000)])
    llrs = llrs.astype(np.float32).astype(np.float64)
    ref_u, _, _ = oracle.scl_batch(llrs, code, 1)
    got = scl_decode_batch(llrs, code, SclConfig(1))
    assert np.array_equal(got.u_hat, ref_u)


def test_noiseless_recovery_all_list_sizes():
    rng = np.random.default_rng(19)
    for N, k in ((8, 4), (64, 40), (1024, 512)):
        code = CodeConfig(N, k, crc=None)
        for L in (1, 2, 4, 8, 32):
            msgs = rng.integers(0, 2, (8, k)).astype(np.uint8)
            x = np.array([polar_transform(insert_message(m, code)) for m in msgs])
            got = scl_decode_batch(channel_llr(modulate_bpsk(x), 0.0), code, SclConfig(L, metric_mode="approx"))
            assert np.array_equal(got.u_hat[:, code.info_positions], msgs)
            assert np.all(got.metric == 0.0)


def test_crc_selected_winner_passes_crc():
    code = CodeConfig(32, 16, crc=8)
    sigma = ebno_to_sigma(1.0, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(31, 0, f))[1] for f in range(300)])
    got = scl_decode_batch(llrs, code, SclConfig(8))
    for f in range(300):
        if got.selected_by_crc[f]:
            assert crc_check(extract_message(got.u_hat[f], code), code.crc)
    assert got.selected_by_crc.sum() > 250


def test_single_frame_api():
    code = CodeConfig(256, 128, crc=16)
    _, llr = make_frame(code, ebno_to_sigma(1.5, code.rate), frame_rng(3, 0, 0))
    llr = llr.astype(np.float32).astype(np.float64)
    r = scl_decode(llr, code, SclConfig(8))
    o = oracle.scl_decode(llr, code, 8)
    assert np.array_equal(r.u_hat, o["u_hat"]) and r.crc_ok == o["crc_ok"]
    with pytest.raises(ValueError):
        scl_decode(np.zeros(8), code)
    bad = np.zeros(256)
    bad[3] = np.inf
    with pytest.raises(ValueError):
        scl_decode(bad, code)


@pytest.mark.parametrize("crc,L", [(24, 8), (8, 32)])
def test_crc_widths_vs_oracle(crc, L):
    """CRC-24 / CRC-8 codes (polar.py:37-41): the incremental syndrome of K3
    against the oracle's CRC-aided winner rule."""
    code = CodeConfig(1024, 700, crc=crc)
    sigma = ebno_to_sigma(2.5, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(2400 + crc, L, f))[1] for f in range(150)])
    llrs = llrs.astype(np.float32).astype(np.float64)
    ref_u, ref_m, ref_ok = oracle.scl_batch(llrs, code, L)
    got = scl_decode_batch(llrs, code, SclConfig(L))
    _compare(f"crc{crc}L{L}", ref_u, ref_m, ref_ok, got)


@pytest.mark.parametrize("N,crc,fmode,mmode,da,B", [
    (64, 8, "minsum", "exact", 0.0, 700), (256, None, "exact", "exact", 0.0, 700),
    (1024, 16, "minsum", "approx", 0.0, 700), (2048, 16, "minsum", "exact", 0.3, 700),
    (2048, 16, "minsum", "exact", 0.0, 3000), (4096, 24, "minsum", "exact", 0.0, 1300)])
def test_sc_kernel_matches_list_kernel_at_l1(N, crc, fmode, mmode, da, B):
    """The SC kernel (sc1.cu: 32/G lanes per frame, element-parallel upper
    levels, speculative decision chain verified by the exact metric rule) is
    bit-identical to K3 v3 at L = 1 (u_hat, metric, CRC flag, payload), in its
    latency form (B <= 8 per SM: one frame per warp) and its throughput form."""
    import os

    import torch

    code = CodeConfig(N, N // 2, crc=crc)
    sigma = ebno_to_sigma(1.5, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(77, N, f))[1] for f in range(B)], dtype=np.float32)
    x = torch.from_numpy(llrs).cuda()
    cfg = SclConfig(1, metric_mode=mmode, f_mode=fmode, da_threshold=da)
    outs = []
    old = os.environ.get("PC_SCL_KERNEL")
    try:
        for kern in ("2", "3"):
            os.environ["PC_SCL_KERNEL"] = kern
            r = scl_decode_batch(x, code, cfg, payload=True)
            torch.cuda.synchronize()
            outs.append((r.u_hat, r.metric, r.crc_ok, r.payload_words))
    finally:
        if old is None:
            os.environ.pop("PC_SCL_KERNEL", None)
        else:
            os.environ["PC_SCL_KERNEL"] = old
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("N,L,eb,count", [(256, 3, 1.5, 300), (256, 5, 1.0, 300), (1024, 6, 1.5, 200),
                                          (1024, 12, 1.5, 150), (512, 20, 1.0, 150), (256, 31, 1.5, 120)])
def test_any_list_size_matches_oracle(N, L, eb, count):
    """The reference accepts any list size (scl.py:57).  A list size that is
    not a power of two runs on the next power of two of lanes with L paths;
    winners, metrics and CRC flags equal the fp64 oracle's (which restates the
    reference's selection for any L)."""
    code = CodeConfig(N, N // 2, crc=16)
    sigma = ebno_to_sigma(eb, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(404, L, f))[1] for f in range(count)])
    llrs = llrs.astype(np.float32).astype(np.float64)
    got = scl_decode_batch(llrs, code, SclConfig(L))
    u, mt, ok = oracle.scl_batch(llrs, code, L)
    assert np.array_equal(got.u_hat, u)
    assert np.array_equal(got.crc_ok, ok)
    assert np.allclose(got.metric, mt, rtol=2e-5, atol=1e-5)


def test_list_size_limits():
    code = CodeConfig(32, 16, crc=None)
    with pytest.raises(ValueError):
        SclConfig(33).native()
    with pytest.raises(ValueError):  # not a power of two and N < 64
        scl_decode_batch(np.zeros((1, 32)), code, SclConfig(3))
