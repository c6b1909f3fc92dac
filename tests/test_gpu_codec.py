"""Encoder / CRC / generator / compaction kernels: bit-exact contracts."""


import numpy as np
import pytest

from conftest import unpack
from paper_1609_09358_b200 import CodeConfig
from paper_1609_09358_b200 import _native as nat
from paper_1609_09358_b200.codes import insert_message, polar_transform

pytestmark = pytest.mark.gpu


def _encode_dev(code, msgs):
    import torch

    dc = nat.device_code(code)
    mw = torch.from_numpy(nat.pack_bits(msgs).view(np.int32)).cuda()
    x = torch.zeros((len(msgs), (code.N + 31) // 32), dtype=torch.int32, device="cuda")
    nat.check(nat.load().pc_encode(mw.data_ptr(), len(msgs), dc.ref, x.data_ptr(), nat.stream_handle()), "encode")
    return nat.unpack_bits(x.cpu().numpy().view(np.uint32), code.N)


def test_encoder_matches_reference_golden(golden):
    code = CodeConfig(1024, 512, crc=16)
    msgs = unpack(golden["enc_msgs"], code.message_len)
    assert np.array_equal(_encode_dev(code, msgs), unpack(golden["enc_x"], 1024))


@pytest.mark.parametrize("N,k,crc", [(8, 4, None), (64, 32, 8), (128, 64, 16), (2048, 1024, 16), (1024, 700, 24)])
def test_encoder_matches_host(N, k, crc):
    code = CodeConfig(N, k, crc=crc)
    rng = np.random.default_rng(N + k)
    msgs = rng.integers(0, 2, (50, code.message_len)).astype(np.uint8)
    ref = np.array([polar_transform(insert_message(m, code)) for m in msgs])
    assert np.array_equal(_encode_dev(code, msgs), ref)


def test_generator_is_consistent_and_keyed():
    import torch

    code = CodeConfig(1024, 512, crc=16)
    dc = nat.device_code(code)
    lib = nat.load()
    B = 256
    MW = (code.message_len + 31) // 32
    msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
    llr = torch.zeros((B, code.N), dtype=torch.float32, device="cuda")
    nat.check(lib.pc_gen_frames(7, 1, 1000, B, 0.0, dc.ref, msg.data_ptr(), llr.data_ptr(), nat.stream_handle()), "gen")
    msgs = nat.unpack_bits(msg.cpu().numpy().view(np.uint32), code.message_len)
    x = (llr.cpu().numpy() < 0).astype(np.uint8)
    assert np.array_equal(x, np.array([polar_transform(insert_message(m, code)) for m in msgs]))
    assert np.all(np.abs(llr.cpu().numpy()) == 20.0)
    assert 0.45 < msgs.mean() < 0.55
    # keyed: frames 1000.. regenerated from frame0 = 1100 overlap exactly
    msg2 = torch.zeros_like(msg)
    llr2 = torch.zeros_like(llr)
    sigma = 0.8
    nat.check(lib.pc_gen_frames(7, 1, 1000, B, sigma, dc.ref, msg.data_ptr(), llr.data_ptr(), nat.stream_handle()), "g")
    nat.check(lib.pc_gen_frames(7, 1, 1100, B, sigma, dc.ref, msg2.data_ptr(), llr2.data_ptr(), nat.stream_handle()), "g")
    assert torch.equal(llr[100:], llr2[:B - 100]) and torch.equal(msg[100:], msg2[:B - 100])
    # noise moments: llr = 2/s^2 (1 - 2x) + (2/s) w
    x = torch.from_numpy(np.array([polar_transform(insert_message(m, code)) for m in
                                   nat.unpack_bits(msg.cpu().numpy().view(np.uint32), code.message_len)]))
    w = (llr.cpu().double() - 2 / sigma**2 * (1 - 2 * x.double())) * sigma / 2
    assert abs(w.mean().item()) < 0.01 and abs(w.std().item() - 1) < 0.01


def test_compaction_is_lossless():
    import torch

    lib = nat.load()
    rng = np.random.default_rng(3)
    for B, p in ((1, 0.5), (1000, 0.1), (100_003, 0.37), (4096, 0.0), (777, 1.0)):
        conv = torch.from_numpy((rng.random(B) > p).astype(np.uint8)).cuda()
        q = torch.full((B,), -1, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        nat.check(lib.pc_compact(conv.data_ptr(), B, q.data_ptr(), cnt.data_ptr(), None, nat.stream_handle()), "c")
        c = int(cnt.item())
        expect = np.flatnonzero(conv.cpu().numpy() == 0)
        assert c == expect.size
        assert np.array_equal(np.sort(q[:c].cpu().numpy()), expect)


def test_error_counter():
    import torch

    rng = np.random.default_rng(4)
    m, B = 496, 300
    a = rng.integers(0, 2, (B, m)).astype(np.uint8)
    b = a.copy()
    flips = rng.random((B, m)) < 0.01
    b[flips] ^= 1
    pa = torch.from_numpy(nat.pack_bits(a).view(np.int32)).cuda()
    pb = torch.from_numpy(nat.pack_bits(b).view(np.int32)).cuda()
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    nat.check(nat.load().pc_count_errors(pa.data_ptr(), pb.data_ptr(), B, m, cnt.data_ptr(), nat.stream_handle()), "e")
    assert cnt[0].item() == flips.sum() and cnt[1].item() == flips.any(axis=1).sum()
