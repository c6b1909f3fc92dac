"""The reference's acceptance claims (pkg/tests/test_acceptance.py, SURVEY.md
section 4) restated for the device path, at sizes the device reaches in
seconds:

* 02: L = 1 equals recursive SC (here: the oracle's L = 1 on 10^4 frames);
* 04: N = 8, k = 4 with L = 16 keeps every path, so the winner is the
  minimum-metric codeword of all 2^k (brute force over the oracle's paths);
* 06: SCL L = 32 beats BP at 2 dB with non-overlapping 95% intervals;
* 07: the hybrid's SCL fallback equals SCL on the failed frames;
* channel: the device generator's uncoded BER equals Q(1/sigma)
  (test_channel.py:84-94 for the host channel).
"""
import math

import numpy as np
import pytest

import oracle
from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig, bp_decode_batch, scl_decode_batch
from paper_1609_09358_b200 import _native as nat
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame
from paper_1609_09358_b200.codes import insert_message, polar_transform

pytestmark = pytest.mark.gpu


def _device_frames(code, eb, B, seed, point=0):
    import torch

    MW = (code.message_len + 31) // 32
    msg = torch.zeros((B, MW), dtype=torch.int32, device="cuda")
    llr = torch.zeros((B, code.N), dtype=torch.float32, device="cuda")
    dc = nat.device_code(code)
    nat.check(nat.load().pc_gen_frames(seed, point, 0, B, ebno_to_sigma(eb, code.rate), dc.ref, msg.data_ptr(),
                                       llr.data_ptr(), nat.stream_handle()), "pc_gen_frames")
    return msg, llr


def _frame_errors(payload_words, msg, m):
    import torch

    MW = (m + 31) // 32
    mask = torch.full((MW,), -1, dtype=torch.int32, device=msg.device)
    if m % 32:
        mask[-1] = (1 << (m % 32)) - 1
    return ((payload_words ^ msg) & mask).ne(0).any(dim=1)


def test_list_size_one_is_sc_on_10k_frames():
    code = CodeConfig(128, 64, crc=None)
    sigma = ebno_to_sigma(2.0, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(2, 0, f))[1] for f in range(10_000)])
    llrs = llrs.astype(np.float32).astype(np.float64)
    got = scl_decode_batch(llrs, code, SclConfig(1))
    ref_u, _, _ = oracle.scl_batch(llrs, code, 1)
    assert np.array_equal(got.u_hat, ref_u)


def test_exhaustive_list_finds_the_minimum_metric_codeword():
    """N=8, k=4, L=16: every one of the 2^k paths survives, so the decoder's
    path list is the whole code and its winner is the global metric minimum."""
    code = CodeConfig(8, 4, crc=None)
    rng = np.random.default_rng(4)
    llrs = (rng.normal(1.0, 1.5, (200, 8))).astype(np.float32).astype(np.float64)
    got = scl_decode_batch(llrs, code, SclConfig(16))
    for f in range(len(llrs)):
        paths, metrics = oracle.scl_paths(llrs[f], code, 16)
        assert len(paths) == 16
        # every codeword appears once
        msgs = {tuple(p[code.info_positions]) for p in paths}
        assert len(msgs) == 16
        best = int(np.lexsort((np.arange(16), metrics))[0])
        assert np.array_equal(got.u_hat[f], paths[best]), f
        assert got.metric[f] == pytest.approx(metrics[best], rel=1e-5, abs=1e-6)


def _wilson(k, n, z=1.96):
    p = k / n
    d = 1 + z * z / n
    c = (p + z * z / (2 * n)) / d
    h = z * math.sqrt(p * (1 - p) / n + z * z / (4 * n * n)) / d
    return c - h, c + h


def test_scl_beats_bp_at_2db_with_separated_intervals():
    code = CodeConfig(1024, 512, crc=16)
    B = 16384
    msg, llr = _device_frames(code, 2.0, B, 606)
    bp = bp_decode_batch(llr, code, BpConfig(stop_mode="crc"), payload=True)
    scl = scl_decode_batch(llr, code, SclConfig(32), payload=True)
    e_bp = int(_frame_errors(bp.payload_words, msg, code.message_len).sum())
    e_scl = int(_frame_errors(scl.payload_words, msg, code.message_len).sum())
    lo_bp, _ = _wilson(e_bp, B)
    _, hi_scl = _wilson(e_scl, B)
    assert hi_scl < lo_bp, (e_scl, e_bp)


def test_hybrid_fallback_equals_scl_on_failed_frames():
    """Frames BP does not converge on get exactly SCL's payload from the
    original LLRs (hybrid.py:131-150); converged frames keep BP's."""
    import torch

    code = CodeConfig(1024, 512, crc=16)
    B = 4096
    _, llr = _device_frames(code, 1.5, B, 707)
    dec = HybridDecoder(code, BpConfig(), SclConfig(32), capacity=B, chunk=1024)
    dec.run(llr).sync()
    hyb = dec.payload[:B].clone()
    conv = dec.conv[:B].bool()
    bp = bp_decode_batch(llr, code, BpConfig(stop_mode="crc"), payload=True)
    scl = scl_decode_batch(llr, code, SclConfig(32), payload=True)
    assert torch.equal(conv, bp.converged)
    assert torch.equal(hyb[conv], bp.payload_words[conv])
    assert torch.equal(hyb[~conv], scl.payload_words[~conv])
    assert 0.05 < (~conv).float().mean().item() < 0.6


@pytest.mark.parametrize("eb", [0.0, 2.0, 4.0])
def test_device_channel_uncoded_ber_is_q_function(eb):
    code = CodeConfig(1024, 512, crc=16)
    B = 4096
    msg, llr = _device_frames(code, eb, B, 808, point=int(eb))
    msgs = nat.unpack_bits(msg.cpu().numpy().view(np.uint32), code.message_len)
    x = np.array([polar_transform(insert_message(m, code)) for m in msgs], dtype=np.uint8)
    hard = (llr.cpu().numpy() < 0).astype(np.uint8)
    ber = float((hard != x).mean())
    sigma = ebno_to_sigma(eb, code.rate)
    q = 0.5 * math.erfc(1.0 / sigma / math.sqrt(2.0))
    n = x.size
    assert abs(ber - q) < 5 * math.sqrt(q * (1 - q) / n) + 1e-6, (ber, q)


def test_throughput_model_eq1_within_25_percent():
    """Reference acceptance test 08 (test_acceptance.py:260-284) on the device
    pipeline, at its exact configuration: N=1024 K=512 CRC-16, L=8, i_max=50,
    768 frames in BP batches of 32, at 1.5 / 2 / 2.5 dB.  The measured
    hybrid_decode_batch throughput must be within 25% of Eq. (1)
    (hybrid.theoretical_throughput) evaluated on the measured BP and SCL
    service rates and gamma."""
    from paper_1609_09358_b200 import FrameJob, hybrid_decode_batch, theoretical_throughput

    assert theoretical_throughput(123.0, 45.0, 0.0) == 123.0
    assert theoretical_throughput(100.0, 1.0, 0.01) == pytest.approx(50.0)
    code = CodeConfig(1024, 512, crc=16)
    gaps = []
    for point, eb in enumerate((1.5, 2.0, 2.5)):
        sigma = ebno_to_sigma(eb, code.rate)
        jobs = []
        for f in range(768):
            m, llr = make_frame(code, sigma, frame_rng(800_000 + point, point, f))
            jobs.append(FrameJob(frame_id=f, llrs=llr, true_message=m))
        kw = dict(bp_batch_size=32, n_scl_workers=2)
        hybrid_decode_batch([FrameJob(frame_id=j.frame_id, llrs=j.llrs, true_message=j.true_message) for j in jobs],
                            code, BpConfig(i_max=50), SclConfig(8), **kw)  # warm-up (allocations, module load)
        st = hybrid_decode_batch(jobs, code, BpConfig(i_max=50), SclConfig(8), **kw)
        gaps.append(abs(st.t_hyb_theo_bps - st.throughput_bps) / st.t_hyb_theo_bps)
    assert max(gaps) < 0.25, f"Eq. (1) gaps {gaps}"
