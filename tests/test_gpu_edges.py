"""Edge cases of the device path against the fp64 oracle: empty batches, the
smallest codes, rate-1 / low-rate codes, ragged batches that do not fill a
warp's frame groups, saturated (noiseless) and all-zero channel LLRs, and the
maximum block length."""
import numpy as np
import pytest

import oracle
from paper_1609_09358_b200 import (BpConfig, CodeConfig, HybridDecoder, SclConfig, bp_decode_batch,
                                   scl_decode_batch)
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame

pytestmark = pytest.mark.gpu


def _frames(code, eb, count, seed):
    sigma = ebno_to_sigma(eb, code.rate)
    x = np.array([make_frame(code, sigma, frame_rng(seed, code.N, f))[1] for f in range(count)])
    return x.astype(np.float32).astype(np.float64)


def test_empty_batches():
    code = CodeConfig(1024, 512, crc=16)
    empty = np.zeros((0, 1024))
    r = bp_decode_batch(empty, code, BpConfig(stop_mode="crc"))
    assert r.u_hat.shape == (0, 1024) and r.converged.shape == (0,)
    s = scl_decode_batch(empty, code, SclConfig(8))
    assert s.u_hat.shape == (0, 1024) and s.metric.shape == (0,)


@pytest.mark.parametrize("N,k,crc", [(2, 1, None), (4, 2, None), (8, 4, None), (16, 16, None), (32, 24, 8),
                                     (64, 20, 16)])
def test_small_and_extreme_rate_codes_scl(N, k, crc):
    """N = 2..64 (the v2 kernel below N = 64, v3 from 64), rate 1 (no frozen
    bit) and low rates: SCL winners equal the oracle's at L = 1, 4, 32."""
    code = CodeConfig(N, k, crc=crc)
    llrs = _frames(code, 1.0, 64, 5)
    for L in (1, 4, 32):
        got = scl_decode_batch(llrs, code, SclConfig(L))
        for f in range(len(llrs)):
            ref = oracle.scl_decode(llrs[f], code, L)
            assert np.array_equal(got.u_hat[f], ref["u_hat"]), (N, k, L, f)
            assert bool(got.crc_ok[f]) == ref["crc_ok"]


@pytest.mark.parametrize("N,k", [(2, 1), (8, 4), (16, 16), (64, 32), (128, 127)])
def test_small_and_extreme_rate_codes_bp(N, k):
    code = CodeConfig(N, k, crc=None)
    llrs = _frames(code, 2.0, 64, 6)
    ref_u, ref_it, ref_cv = oracle.bp_batch(llrs, code, i_max=20, stop_mode="reencode")
    got = bp_decode_batch(llrs, code, BpConfig(i_max=20, stop_mode="reencode"))
    same = (got.iterations_used == ref_it) & (got.converged == ref_cv)
    assert same.mean() >= 0.97, np.flatnonzero(~same)
    for f in np.flatnonzero(same & ref_cv):
        assert np.array_equal(got.u_hat[f], ref_u[f])


@pytest.mark.parametrize("L,B", [(2, 17), (4, 13), (8, 5), (16, 3), (1, 33)])
def test_ragged_batches_fill_partial_frame_groups(L, B):
    """B not a multiple of the 32/L frames one warp decodes: the idle groups
    must not disturb the live ones."""
    code = CodeConfig(1024, 512, crc=16)
    llrs = _frames(code, 1.5, B, 7)
    got = scl_decode_batch(llrs, code, SclConfig(L))
    ref_u, _, ref_ok = oracle.scl_batch(llrs, code, L)
    assert np.array_equal(got.u_hat, ref_u) and np.array_equal(got.crc_ok, ref_ok)


def test_saturated_and_zero_llrs():
    """Noiseless +-20 LLRs decode in one BP iteration and to the right path;
    all-zero LLRs (no channel information) follow the reference's tie rules
    (an exact 0 decides bit 0; SCL ties by candidate index)."""
    code = CodeConfig(256, 128, crc=16)
    sat = np.full((4, 256), 20.0)  # the all-zero codeword
    r = bp_decode_batch(sat, code, BpConfig(stop_mode="crc"))
    assert r.converged.all() and (r.iterations_used == 1).all() and not r.u_hat.any()
    zero = np.zeros((3, 256))
    rb = bp_decode_batch(zero, code, BpConfig(i_max=5, stop_mode="none"))
    ref = oracle.bp_decode(zero[0], code, i_max=5, stop_mode="none")
    assert np.array_equal(rb.u_hat[0], ref["u_hat"])
    for L in (1, 8, 32):
        s = scl_decode_batch(zero, code, SclConfig(L))
        o = oracle.scl_decode(zero[0], code, L)
        assert np.array_equal(s.u_hat[0], o["u_hat"]) and s.metric[0] == pytest.approx(o["metric"], rel=1e-5)


def test_maximum_block_length_hybrid_chunks():
    """N = 4096 through the hybrid pipeline in ragged chunks (the last chunk
    partial) against the oracle's hybrid on the same fp32 LLRs."""
    code = CodeConfig(4096, 2048, crc=16)
    llrs = _frames(code, 1.5, 40, 8)
    import torch

    dec = HybridDecoder(code, BpConfig(), SclConfig(8), capacity=64, chunk=16)
    dec.run(torch.from_numpy(llrs.astype(np.float32)).cuda()).sync()
    got = dec.host_results()
    pay, prov, _ = oracle.hybrid_batch(llrs, code, L=8)
    words = got["payload"]
    bits = ((words[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(len(llrs), -1)[:, :code.message_len]
    agree = (bits == pay).all(axis=1)
    # frames may part only where BP provenance flips on a near-tie (test_gpu_hybrid.py)
    assert agree.mean() >= 0.95, np.flatnonzero(~agree)


def test_tampered_first_info_is_refused_not_decoded():
    """A reference-side binding that sets pc_code_t.first_info past info_pos[0]
    gets PC_ERR_INVALID from pc_scl_decode (the struct's seal no longer
    matches), not silently wrong decisions; pc_code_seal derives the right
    value and rejects tables that contradict each other."""
    import ctypes

    import torch

    from paper_1609_09358_b200 import _native as nat

    code = CodeConfig(1024, 512, crc=16)
    dc = nat.device_code(code)
    assert dc.struct.first_info == int(code.info_positions[0]) == 191
    lib = nat.load()
    cfg = SclConfig(32).native()
    llr = torch.ones((1, 1024), dtype=torch.float32, device="cuda")
    u = torch.zeros((1, 32), dtype=torch.int32, device="cuda")
    ws = dc.new_scl_workspace(cfg)
    bad = nat.PcCode.from_buffer_copy(dc.struct)
    bad.first_info = 224
    rc = lib.pc_scl_decode(llr.data_ptr(), 1, None, None, ctypes.byref(bad), ctypes.byref(cfg), u.data_ptr(), None,
                           None, None, None, None, ws.data_ptr(), nat.stream_handle())
    assert rc == -1
    # resealing derives first_info from the tables again
    assert lib.pc_code_seal(ctypes.byref(bad), nat.stream_handle()) == 0 and bad.first_info == 191
    assert lib.pc_scl_decode(llr.data_ptr(), 1, None, None, ctypes.byref(bad), ctypes.byref(cfg), u.data_ptr(),
                             None, None, None, None, None, ws.data_ptr(), nat.stream_handle()) == 0
    # info_pos that is not the ascending list of non-frozen positions is rejected
    ip = dc.info_pos.clone()
    ip[[0, 1]] = ip[[1, 0]]
    wrong = nat.PcCode.from_buffer_copy(dc.struct)
    wrong.info_pos = ip.data_ptr()
    assert lib.pc_code_seal(ctypes.byref(wrong), nat.stream_handle()) == -1
    fz = dc.frozen_bits.clone()
    fz[0] ^= 1
    wrong = nat.PcCode.from_buffer_copy(dc.struct)
    wrong.frozen_bits = fz.data_ptr()
    assert lib.pc_code_seal(ctypes.byref(wrong), nat.stream_handle()) == -1
    torch.cuda.synchronize()
