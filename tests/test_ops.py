"""The PyTorch extension (paper_1609_09358_b200/ops.py, csrc/torch_ops.cpp):
the op library loads and registers its ops and class on a CPU host; on the
B200 its results equal the package's batch APIs bit for bit."""

import numpy as np
import pytest

from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig, bp_decode_batch, scl_decode_batch
from paper_1609_09358_b200 import ops
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame


def test_op_library_registers_ops():
    import torch

    polar = ops.load()
    for name in ("bp_decode", "scl_decode", "hybrid_decode", "gen_frames", "encode"):
        assert hasattr(polar, name)
    assert torch.classes.polar.Code is not None


def _frames(code, eb, B, seed):
    import torch

    sigma = ebno_to_sigma(eb, code.rate)
    x = np.array([make_frame(code, sigma, frame_rng(seed, code.N, f))[1] for f in range(B)], dtype=np.float32)
    return torch.from_numpy(x).cuda()


@pytest.mark.gpu
@pytest.mark.parametrize("N,mode", [(128, "crc"), (1024, "reencode"), (2048, "crc")])
def test_bp_op_equals_batch_api(N, mode):
    import torch

    code = CodeConfig(N, N // 2, crc=16)
    x = _frames(code, 2.0, 300, 5)
    cfg = BpConfig(i_max=30, stop_mode=mode)
    u, pay, it, cv, su, sx = ops.bp_decode(x, code, cfg, soft=True)
    ref = bp_decode_batch(x, code, cfg)
    torch.cuda.synchronize()
    assert torch.equal(it, ref.iterations_used) and torch.equal(cv.bool(), ref.converged.bool())
    assert torch.equal(u, ref.u_hat)


@pytest.mark.gpu
@pytest.mark.parametrize("N,L", [(256, 1), (1024, 32), (512, 6)])
def test_scl_op_equals_batch_api(N, L):
    import torch

    code = CodeConfig(N, N // 2, crc=16)
    x = _frames(code, 1.5, 200, 6)
    u, pay, mt, ok, sel = ops.scl_decode(x, code, SclConfig(L))
    ref = scl_decode_batch(x, code, SclConfig(L), payload=True)
    torch.cuda.synchronize()
    assert torch.equal(u, ref.u_hat) and torch.equal(mt, ref.metric) and torch.equal(pay, ref.payload_words)
    assert torch.equal(ok.bool(), ref.crc_ok.bool())


@pytest.mark.gpu
def test_hybrid_op_equals_decoder():
    import torch

    code = CodeConfig(1024, 512, crc=16)
    x = _frames(code, 1.5, 500, 7)
    pay, cv, it = ops.hybrid_decode(x, code, BpConfig(), SclConfig(32))
    dec = HybridDecoder(code, BpConfig(), SclConfig(32), capacity=500)
    dec.run(x).sync()
    torch.cuda.synchronize()
    assert torch.equal(pay, dec.payload[:500]) and torch.equal(cv, dec.conv[:500]) and torch.equal(it, dec.iters[:500])
    assert int((cv == 0).sum()) > 50


@pytest.mark.gpu
def test_gen_frames_op_equals_abi():
    import torch

    from paper_1609_09358_b200 import _native as nat

    code = CodeConfig(512, 256, crc=16)
    msg, llr = ops.gen_frames(code, 11, 2, 100, 64, 0.8)
    dc = nat.device_code(code)
    m2 = torch.zeros_like(msg)
    l2 = torch.zeros_like(llr)
    nat.check(nat.load().pc_gen_frames(11, 2, 100, 64, 0.8, dc.ref, m2.data_ptr(), l2.data_ptr(),
                                       nat.stream_handle()), "gen")
    torch.cuda.synchronize()
    assert torch.equal(msg, m2) and torch.equal(llr, l2)
