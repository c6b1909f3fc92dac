"""World-size-2 gloo test of the frame sharding (CPU): two ranks decode their
shards with the CPU oracle as a stand-in decoder, merge counters with the
same helpers bench.py uses, and must reproduce the single-process counts."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1609_09358_b200 import CodeConfig
from paper_1609_09358_b200.shard import COUNTER_FIELDS, merge_counters, shard_range, split_total

PER_RANK = 24
EBNO = 1.5


def _count(lo, hi):
    import oracle
    from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame

    code = CodeConfig(256, 128, crc=16)
    sigma = ebno_to_sigma(EBNO, code.rate)
    fr = [make_frame(code, sigma, frame_rng(7, 0, f)) for f in range(lo, hi)]
    msgs = np.array([f[0] for f in fr])
    llrs = np.array([f[1] for f in fr])
    pay, prov, iters = oracle.hybrid_batch(llrs, code, i_max=20, L=4, nthreads=2)
    errs = (pay != msgs).sum(axis=1)
    return {"frames": hi - lo, "bit_errors": int(errs.sum()), "frame_errors": int((errs > 0).sum()),
            "frames_to_scl": int(prov.sum()), "bp_iterations": int(iters.sum())}


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(rank, world, PER_RANK)
    merged = merge_counters(_count(lo, hi))
    q.put((rank, merged))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_shards_reproduce_single_process_counts():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = _count(0, 2 * PER_RANK)
    assert results[0] == results[1] == {k: single[k] for k in COUNTER_FIELDS}


def test_shard_ranges_partition():
    assert shard_range(0, 2, 10) == (0, 10) and shard_range(1, 2, 10) == (10, 20)
    parts = split_total(103, 4)
    assert parts[0][0] == 0 and parts[-1][1] == 103
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    with pytest.raises(ValueError):
        shard_range(2, 2, 10)


# ---------------------------------------------------------------- device --
def _count_device(lo, hi):
    """Device hybrid pipeline (K1 -> K2 -> K3) over global frames [lo, hi)."""
    import torch

    from paper_1609_09358_b200 import BpConfig, HybridDecoder, SclConfig
    from paper_1609_09358_b200 import _native as nat
    from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame

    torch.cuda.set_device(0)
    code = CodeConfig(256, 128, crc=16)
    sigma = ebno_to_sigma(EBNO, code.rate)
    fr = [make_frame(code, sigma, frame_rng(7, 0, f)) for f in range(lo, hi)]
    msgs = np.array([f[0] for f in fr])
    llrs = np.array([f[1] for f in fr]).astype(np.float32)
    dec = HybridDecoder(code, BpConfig(i_max=20), SclConfig(4), capacity=hi - lo, chunk=16)
    dec.run(torch.from_numpy(llrs).cuda()).sync()
    r = dec.host_results()
    errs = (nat.unpack_bits(r["payload"], code.message_len) != msgs).sum(axis=1)
    return {"frames": hi - lo, "bit_errors": int(errs.sum()), "frame_errors": int((errs > 0).sum()),
            "frames_to_scl": int((~r["converged"]).sum()), "bp_iterations": int(r["iters"].sum())}


def _worker_device(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(rank, world, PER_RANK)
    merged = merge_counters(_count_device(lo, hi))
    q.put((rank, merged))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_device_shards_reproduce_single_process_counts():
    """The product path under two ranks (both on cuda:0 of the one-GPU box,
    counters merged over gloo) equals one process decoding all the frames."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_device, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = _count_device(0, 2 * PER_RANK)
    assert results[0] == results[1] == {k: single[k] for k in COUNTER_FIELDS}
