"""Hybrid pipeline (K1 -> K2 -> K3 on two streams) parity and bookkeeping."""

import math

import numpy as np
import pytest

import oracle
from conftest import golden_frames, unpack
from paper_1609_09358_b200 import (
    BpConfig,
    CodeConfig,
    FrameJob,
    HybridDecoder,
    SclConfig,
    hybrid_decode_batch,
    hybrid_decode_frame,
    latency_stats,
    theoretical_throughput,
)
from paper_1609_09358_b200 import _native as nat
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["hyb1024a", "hyb1024b"])
def test_hybrid_frames_match_reference(golden, golden_meta, name):
    meta = golden_meta["sets"][name]
    code = CodeConfig(1024, 512, crc=16)
    _, llrs = golden_frames(meta, code)
    ref_pay = unpack(golden[f"{name}_payload"], code.message_len)
    ref_scl = golden[f"{name}_scl"]
    jobs = [FrameJob(frame_id=f, llrs=llrs[f]) for f in range(len(llrs))]
    hybrid_decode_batch(jobs, code, BpConfig(i_max=50), SclConfig(32), bp_batch_size=16)
    bad = [f for f, j in enumerate(jobs) if not np.array_equal(j.message, ref_pay[f])
           or (j.provenance == "scl") != bool(ref_scl[f])]
    assert len(bad) <= 1, f"{name}: {bad}"
    p, prov = hybrid_decode_frame(llrs[0], code, BpConfig(i_max=50), SclConfig(32))
    assert np.array_equal(p, ref_pay[0]) and (prov == "scl") == bool(ref_scl[0])


def test_device_pipeline_vs_oracle_hybrid():
    """3000 frames at 1.5 dB through HybridDecoder (chunked, overlapped) vs the C oracle.

    Every payload difference must come from a BP provenance flip on a near-tie
    frame (reference BP still iterating past 20 iterations); the error counts
    against the true payload must be statistically indistinguishable (paired
    sign test on discordant frames, as reference test_acceptance.py:223-257).
    """
    import torch

    code = CodeConfig(1024, 512, crc=16)
    sigma = ebno_to_sigma(1.5, code.rate)
    fr = [make_frame(code, sigma, frame_rng(2024, 2, f)) for f in range(3000)]
    msgs = np.array([f[0] for f in fr])
    llrs = np.array([f[1] for f in fr]).astype(np.float32).astype(np.float64)
    pay, prov, iters = oracle.hybrid_batch(llrs, code, i_max=50, L=32)
    dec = HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=3000, chunk=512)
    dec.run(torch.from_numpy(llrs.astype(np.float32)).cuda()).sync()
    r = dec.host_results()
    got = nat.unpack_bits(r["payload"], code.message_len)
    dev_scl = ~r["converged"]
    diff = np.flatnonzero((got != pay).any(axis=1))
    flips = np.flatnonzero(dev_scl != prov)
    print(f"gamma={dev_scl.mean():.3f} provenance flips={flips.size} payload diffs={diff.size}")
    assert set(diff.tolist()) <= set(flips.tolist()), "payload differs on a frame both sides routed alike"
    assert np.all(iters[flips] > 20), "provenance flip on a frame the reference decided early"
    assert flips.size <= 0.02 * len(llrs)
    assert r["counts"].sum() == dev_scl.sum()  # no frame lost by the compaction
    dev_err = (got != msgs).any(axis=1)
    ref_err = (pay != msgs).any(axis=1)
    a, b = int((dev_err & ~ref_err).sum()), int((ref_err & ~dev_err).sum())
    if a + b:
        p = min(1.0, sum(math.comb(a + b, i) for i in range(min(a, b) + 1)) / 2 ** (a + b - 1))
        assert p > 0.01, f"paired error test rejects equality (dev-only {a}, ref-only {b})"


def _jobs(code, sigma, count, seed):
    out = []
    for f in range(count):
        msg, llr = make_frame(code, sigma, frame_rng(seed, 0, f))
        out.append(FrameJob(frame_id=f, llrs=llr, true_message=msg))
    return out


def test_batch_bookkeeping():
    code = CodeConfig(64, 32, crc=8)
    jobs = _jobs(code, 1.2, 40, 7)
    stats = hybrid_decode_batch(jobs, code, BpConfig(i_max=5), SclConfig(4), bp_batch_size=8)
    assert stats.frames_total == 40 and stats.info_bits == 40 * code.message_len
    assert stats.frames_to_scl == sum(j.status == "scl_done" for j in jobs)
    assert stats.gamma_bp_fer == pytest.approx(stats.frames_to_scl / 40)
    assert stats.overhead_s == pytest.approx(stats.wall_s - stats.bp_busy_s - stats.scl_busy_s)
    lat = latency_stats(jobs)
    assert stats.latency_avg_s == pytest.approx(lat["hybrid_avg_s"])
    if stats.frames_to_scl:
        assert stats.t_hyb_theo_bps == pytest.approx(
            theoretical_throughput(stats.t_bp_bps, stats.t_scl_bps, stats.gamma_bp_fer))
    for j in jobs:
        if j.provenance == "scl":
            assert j.t_scl_end >= j.t_scl_start >= j.t_bp_end >= j.t_enqueue
        else:
            assert math.isnan(j.t_scl_end)
    for base in range(0, 40, 8):
        batch = jobs[base:base + 8]
        assert len({j.t_enqueue for j in batch}) == 1 and len({j.t_bp_end for j in batch}) == 1


def test_batch_all_converged_and_noiseless():
    code = CodeConfig(64, 32, crc=8)
    jobs = _jobs(code, 0.0, 24, 9)
    stats = hybrid_decode_batch(jobs, code, bp_batch_size=8)
    assert stats.frames_to_scl == 0 and math.isnan(stats.t_scl_bps)
    assert stats.t_hyb_theo_bps == stats.t_bp_bps
    for j in jobs:
        assert j.provenance == "bp" and np.array_equal(j.message, j.true_message)


def test_validation():
    code = CodeConfig(32, 16, crc=8)
    with pytest.raises(ValueError):
        hybrid_decode_batch([], code)
    with pytest.raises(ValueError):
        hybrid_decode_batch([FrameJob(0, np.zeros(32))], code, bp_batch_size=0)
    with pytest.raises(ValueError):
        hybrid_decode_batch([FrameJob(0, np.zeros(16))], CodeConfig(16, 8, crc=None))


def test_host_buffer_pipeline_matches_device_run():
    """decode_host_many (H2D of batch i+1 overlapping the decode of batch i)
    returns exactly what run() produces batch by batch."""
    import torch

    code = CodeConfig(1024, 512, crc=16)
    batches = []
    for p, eb in enumerate((1.0, 2.0, 3.0)):
        sigma = ebno_to_sigma(eb, code.rate)
        llrs = np.array([make_frame(code, sigma, frame_rng(55, p, f))[1] for f in range(300 + 50 * p)])
        batches.append(torch.from_numpy(llrs.astype(np.float32)).pin_memory())
    dec = HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=400, chunk=128)
    got = dec.decode_host_many(batches)
    for b, (pay, conv) in zip(batches, got):
        dec.run(b.cuda(), b.shape[0]).sync()
        r = dec.host_results()
        assert np.array_equal(pay, r["payload"]) and np.array_equal(conv, r["converged"])


def test_n4096_hybrid_vs_oracle():
    """C4's code through the whole hybrid (K1 at N=4096, K3 at N=4096 L=32)."""
    import torch

    code = CodeConfig(4096, 2048, crc=16)
    sigma = ebno_to_sigma(2.0, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(4097, 0, f))[1] for f in range(96)])
    llrs = llrs.astype(np.float32).astype(np.float64)
    pay, prov, iters = oracle.hybrid_batch(llrs, code, i_max=50, L=32)
    dec = HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=96, chunk=48)
    dec.run(torch.from_numpy(llrs.astype(np.float32)).cuda()).sync()
    r = dec.host_results()
    got = nat.unpack_bits(r["payload"], code.message_len)
    flips = np.flatnonzero(~r["converged"] != prov)
    diff = np.flatnonzero((got != pay).any(axis=1))
    assert (~r["converged"]).sum() > 0, "no frame reached the list decoder"
    assert set(diff.tolist()) <= set(flips.tolist())
    assert np.all(iters[flips] > 20) and flips.size <= 2


def test_results_do_not_depend_on_chunking():
    """Per-frame outputs are independent of the chunk size (ragged last chunk,
    per-chunk queues and counters), of the stream overlap and of the number
    of SCL streams (concurrent K3 launches on their own workspaces)."""
    import torch

    code = CodeConfig(1024, 512, crc=16)
    sigma = ebno_to_sigma(1.5, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(77, 0, f))[1] for f in range(1000)])
    x = torch.from_numpy(llrs.astype(np.float32)).cuda()
    ref = None
    for chunk, overlap, ns in ((1000, True, None), (333, True, None), (100, False, None), (1, True, None),
                               (32, True, 1), (32, True, 3), (32, True, 8)):
        dec = HybridDecoder(code, BpConfig(i_max=50), SclConfig(32), capacity=1000, chunk=chunk, overlap=overlap,
                            scl_streams=ns)
        dec.run(x).sync()
        r = dec.host_results()
        assert r["counts"].sum() == (~r["converged"]).sum()
        if ref is None:
            ref = r
        else:
            assert np.array_equal(r["payload"], ref["payload"]) and np.array_equal(r["converged"], ref["converged"])
            assert np.array_equal(r["iters"], ref["iters"])


def test_scl_queue_subset_and_empty_queue():
    """K3 decodes exactly the queued frames (others untouched) and a zero-length
    queue launches nothing."""
    import ctypes
    import torch

    code = CodeConfig(1024, 512, crc=16)
    sigma = ebno_to_sigma(1.5, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(78, 0, f))[1] for f in range(64)])
    x = torch.from_numpy(llrs.astype(np.float32)).cuda()
    from paper_1609_09358_b200 import scl_decode_batch

    full = scl_decode_batch(x, code, SclConfig(32), payload=True)
    lib = nat.load()
    dc = nat.device_code(code)
    cfg = SclConfig(32).native()
    MW = (code.message_len + 31) // 32
    for q in ([5, 17, 40, 63], []):
        queue = torch.tensor(q + [0], dtype=torch.int32, device="cuda")
        count = torch.tensor([len(q)], dtype=torch.int32, device="cuda")
        pay = torch.full((64, MW), -1, dtype=torch.int32, device="cuda")
        nat.check(lib.pc_scl_decode(x.data_ptr(), 64, queue.data_ptr(), count.data_ptr(), dc.ref, ctypes.byref(cfg),
                                    None, pay.data_ptr(), None, None, None, None,
                                    dc.scl_workspace(cfg).data_ptr(), nat.stream_handle()), "scl")
        p = pay.cpu().numpy()
        for f in range(64):
            if f in q:
                assert np.array_equal(p[f], full.payload_words[f].cpu().numpy())
            else:
                assert np.all(p[f] == -1)


@pytest.mark.parametrize("L", [1, 6])
def test_hybrid_any_list_size_vs_oracle(L):
    """The hybrid with a list size that is not a power of two (L = 6: the list
    decoder keeps 6 paths on 8 lanes) and with L = 1 (the SC kernel on the
    queue of BP failures): payloads equal the oracle's on every frame both
    sides route alike."""
    import torch

    code = CodeConfig(1024, 512, crc=16)
    sigma = ebno_to_sigma(1.5, code.rate)
    llrs = np.array([make_frame(code, sigma, frame_rng(2025, L, f))[1] for f in range(800)])
    llrs = llrs.astype(np.float32).astype(np.float64)
    pay, prov, iters = oracle.hybrid_batch(llrs, code, i_max=50, L=L)
    dec = HybridDecoder(code, BpConfig(i_max=50), SclConfig(L), capacity=800, chunk=256)
    dec.run(torch.from_numpy(llrs.astype(np.float32)).cuda()).sync()
    r = dec.host_results()
    got = nat.unpack_bits(r["payload"], code.message_len)
    flips = np.flatnonzero(~r["converged"] != prov)
    diff = np.flatnonzero((got != pay).any(axis=1))
    assert set(diff.tolist()) <= set(flips.tolist())
    assert np.all(iters[flips] > 20) and flips.size <= 0.02 * len(llrs)
    assert (~r["converged"]).sum() > 100  # the list decoder ran on a real queue


def test_graph_replay_matches_eager_run():
    """run(graph=True): the first call runs eagerly and captures the whole
    pipeline (chunks on the BP and SCL streams) as a CUDA graph; replays give
    the eager results, for new contents of the same input buffer too."""
    import torch

    code = CodeConfig(1024, 512, crc=16)
    sigma = ebno_to_sigma(1.5, code.rate)
    frames = [np.array([make_frame(code, sigma, frame_rng(79 + k, 0, f))[1] for f in range(300)]) for k in range(2)]
    x = torch.empty((300, 1024), device="cuda")
    eager = HybridDecoder(code, BpConfig(i_max=50), SclConfig(8), capacity=300, chunk=32)
    dec = HybridDecoder(code, BpConfig(i_max=50), SclConfig(8), capacity=300, chunk=32)
    for k in range(2):
        x.copy_(torch.from_numpy(frames[k].astype(np.float32)))
        ref = eager.run(x).sync().host_results()
        for _ in range(2):  # capture (eager), then replay
            dec.payload.zero_()
            dec.conv.zero_()
            r = dec.run(x, graph=True).sync().host_results()
            for key in ("payload", "converged", "iters", "counts"):
                assert np.array_equal(r[key], ref[key]), key
    assert len(dec._graphs) == 1
