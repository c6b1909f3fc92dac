#!/usr/bin/env python
"""Headline benchmark: hybrid BP -> SCL decoding, N=1024 K=512 (496 payload +
16 CRC bits), L=32, i_max=50, swept over Eb/N0 = 1..4 dB (BASELINE.json).

A step = one pass of the device pipeline (K1 BP with fused CRC stop -> K2
compaction -> K3 CRC-aided SCL on the failures) over one batch of B frames at
EVERY sweep point.  value = decoded payload Gbit/s over the whole sweep
(sum of bits / sum of time), whole job over all ranks; per-point Gbit/s, p50
frame latency, gamma and FER are in "sweep".

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python bench.py --workload c1     # BASELINE configs[0]: BP N=128, 2 dB
    python bench.py --workload c2     # BASELINE configs[1]: SCL N=1024 L=32, 1-4 dB
    python bench.py --workload c4     # BASELINE configs[3]: large-batch BP N=4096, 2 and 3 dB
    python bench.py --workload c5     # BASELINE configs[4]: SCL N=2048 list-size sweep L=1..32

The default workload (c3) is the headline; the others print their own JSON
line (same contract keys) for the other BASELINE configurations.  c3 times
the points one after another (value, roofline and shares come from that
region) and then the same steps with the cross-point overlap ("overlapped");
"e2e" runs the public host-buffer call; "parity_sample" decodes the
cpu_baseline frames on the device beside the oracle's results.

Multi-GPU: frames shard by index (weak scaling, no collective on the data
path); timing is the max over ranks of the barrier-bracketed device time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decoded info Gbit/s, hybrid BP+SCL N=1024 L=32, vs Eb/N0; p50 frame latency"
EBNO = (1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0)
N, K, LIST, IMAX = 1024, 512, 32, 50
SEED = 20240917
def mufu_per_alg_g(n: int) -> float:
    """MUFU ops K1 spends per ALGORITHMIC exact g (the reference's 2nN per
    frame-iteration, bp.py:138-161).  K1 runs the likelihood-ratio form
    (bp_math.cuh, g_mode 0): one MUFU.RCP per g, and R[n] (never read) is not
    computed, so a frame-iteration is (2n - 1) N/2 PEs x 2 RCP."""
    return (2 * n - 1) / (2 * n)


def k1_tpf(N: int) -> int:
    """K1's default threads per frame for the likelihood-ratio form: Q = 8
    nodes per thread (bp3.cu from N = 256, bp3h.cu at N = 128: a half-warp)."""
    return N // 8


def _clock_mhz(ck):
    peak_mhz = 1965.0
    try:
        peak_mhz = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("sm_max_mhz", 1965.0))
    except Exception:
        pass
    return (ck or {}).get("sm_mhz") or peak_mhz, peak_mhz


def k1_kernel_label(N: int) -> str:
    n = N.bit_length() - 1
    if N >= 256:
        return (f"k_bp3<{n},0> (BP, likelihood-ratio arithmetic, {N // 8} threads/frame, warp-local boundaries in "
                "three register layouts joined by shared-memory transposes)")
    if N == 128:
        return ("k_bp3h<0> (BP, likelihood-ratio arithmetic, a frame per half-warp, 7 boundaries in three register "
                "layouts joined by shared-memory transposes)")
    return f"k_bp2<{n},{max(32, N // 8)},0> (BP, likelihood-ratio arithmetic, lane-pair shuffles, one warp per frame)"


def k1_roofline(torch, dev, N: int, g_total: float, k1_s: float, ck, frames_per_launch=None) -> dict:
    """Roofline of K1 from live numbers: g_total algorithmic exact-g
    evaluations (sum of iterations x 2nN) in k1_s seconds of K1 time (CUDA
    events on K1's stream).  HBM is < 1% (4.2 KB per frame), so the bound is
    an SM pipe.  Two are computed and the LOWER one is `peak` (`bound`):
      * xu: the MUFU pipe, 148 SM x 16/clk at the measured SM clock, divided by
        K1's MUFU per algorithmic g (one RCP per g of the likelihood-ratio
        form, R[n] not computed: (2n-1)/(2n));
      * issue: 148 SM x 4 warp-instructions/clk divided by the
        warp-instructions K1 executes per algorithmic g (one ncu capture of the
        same kernel, profiles/k1_issue.json).
    `frac_alg` is SURVEY.md section 8(d)'s fixed formula (achieved x 4 MUFU per
    g / XU peak), which the likelihood-ratio arithmetic exceeds by design."""
    n = N.bit_length() - 1
    achieved = g_total / k1_s / 1e9
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz, max_mhz = _clock_mhz(ck)
    xu_ops = sms * 16 * mhz * 1e6
    mpg = mufu_per_alg_g(n)
    xu_peak = xu_ops / mpg / 1e9
    issue = None
    try:
        issue = json.loads((ROOT / "profiles" / "k1_issue.json").read_text())[str(N)]
    except Exception:
        pass
    ipg = issue["warp_inst_per_alg_g"] if issue else None
    issue_peak = sms * 4 * mhz * 1e6 / ipg / 1e9 if ipg else None
    bound, peak = ("xu", xu_peak) if issue_peak is None or xu_peak <= issue_peak else ("issue", issue_peak)
    traffic = None
    try:
        per_frame = json.loads((ROOT / "profiles" / "bp_kernel_ncu.json").read_text())["dram_bytes_per_frame"]
        if N == 1024 and frames_per_launch:
            traffic = per_frame * frames_per_launch
    except Exception:
        pass
    return {
        "bound": bound, "achieved": achieved, "peak": peak, "unit": "Gg/s", "frac": achieved / peak,
        "traffic": traffic, "frac_alg": achieved * 4 / (xu_ops / 1e9), "kernel": k1_kernel_label(N),
        "sm_mhz": mhz, "sm_max_mhz": max_mhz,
        "xu": {"mufu_per_alg_g": mpg, "peak": xu_peak, "frac": achieved / xu_peak},
        "issue": {"warp_inst_per_alg_g": ipg, "peak": issue_peak,
                  "frac": achieved / issue_peak if issue_peak else None,
                  "source": issue.get("source") if issue else None},
        "note": "unit = one exact-g evaluation as the reference counts them (2nN per frame-iteration, "
                "bp.py:138-161); peak = the lower of the MUFU (xu) and instruction-issue bounds at the measured "
                "SM clock; frac_alg = SURVEY 8(d)'s XU formula at 4 MUFU per g; HBM < 1% (4.2 KB per frame)",
    }


WORKLOAD = "hybrid BP->SCL N=1024 K=512 (496 payload + CRC-16) L=32 i_max=50, Eb/N0 1-4 dB step 0.5"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def spawn_ranks(n: int) -> int:
    """``--gpus N`` without a launcher: re-run this script as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1).
    Rank 0 prints the JSON line; torchrun's exit code is returned."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 7:
                    self.rows.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------ CPU baseline --
_CPU_FRAMES: dict = {}
# tools/ref_vs_port.py (8-core dev container, 256 frames per point, payloads identical)
try:
    PORT_OVER_REF = json.loads((ROOT / "profiles" / "ref_vs_port.json").read_text())["port_over_reference"]
except Exception:
    PORT_OVER_REF = float("nan")


def cpu_hybrid_sample(frames_per_point: int, threads: int, keep: dict | None = None):
    """The oracle port (oracle/oracle.c, fp64, the reference's algorithm) on the
    host cores over a bounded sample of the same sweep; returns (Gbit/s, busy
    seconds).  The frames are host PCG64 frames with fp32-rounded LLRs (what the
    device decodes); with ``keep`` the oracle's payloads and provenance per point
    are stored there for the parity sample."""
    import oracle
    from paper_1609_09358_b200 import CodeConfig
    from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame

    code = CodeConfig(N, K, crc=16)
    bits = 0
    busy = 0.0
    for p, eb in enumerate(EBNO):
        key = (p, frames_per_point)
        if key not in _CPU_FRAMES:  # host PCG64 frames, generated once per (point, size)
            sigma = ebno_to_sigma(eb, code.rate)
            fr = [make_frame(code, sigma, frame_rng(SEED, p, f)) for f in range(frames_per_point)]
            _CPU_FRAMES[key] = (np.array([f[0] for f in fr]),
                                np.array([f[1] for f in fr]).astype(np.float32).astype(np.float64))
        msgs, llrs = _CPU_FRAMES[key]
        t0 = time.perf_counter()
        pay, prov, _ = oracle.hybrid_batch(llrs, code, i_max=IMAX, L=LIST, nthreads=threads)
        busy += time.perf_counter() - t0
        bits += frames_per_point * code.message_len
        if keep is not None:
            keep[p] = (msgs, llrs, pay, prov)
    return bits / busy / 1e9, busy


def parity_sample(torch, dev, keep: dict) -> dict:
    """The cpu_baseline sample's frames decoded by the device pipeline beside
    the oracle's results on the same fp32 LLRs: identical payloads, BP/SCL
    provenance flips (fp32 vs fp64 near-ties in BP) and the
    frame errors of both (whose equality in distribution is the parity
    criterion, tests/parity/fer_parity*.py)."""
    from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig
    from paper_1609_09358_b200 import _native as nat

    code = CodeConfig(N, K, crc=16)
    m = code.message_len
    n = max(v[1].shape[0] for v in keep.values())
    d = HybridDecoder(code, BpConfig(i_max=IMAX), SclConfig(LIST), capacity=n, device=dev)
    tot = same = flips = fe_dev = fe_ref = 0
    for p in sorted(keep):
        msgs, llrs, pay, prov = keep[p]
        x = torch.from_numpy(llrs.astype(np.float32)).to(dev)
        r = d.run(x).sync().host_results()
        got = nat.unpack_bits(r["payload"], m)
        tot += len(msgs)
        same += int(np.all(got == pay, axis=1).sum())
        flips += int(((~r["converged"]) != prov.astype(bool)).sum())
        fe_dev += int(np.any(got != msgs, axis=1).sum())
        fe_ref += int(np.any(pay != msgs, axis=1).sum())
    return {"frames": tot, "payload_identical": same, "provenance_flips": flips, "frame_errors_device": fe_dev,
            "frame_errors_oracle": fe_ref,
            "note": "the cpu_baseline frames (host PCG64, fp32-rounded LLRs) through the device pipeline vs the "
                    "fp64 oracle port of the reference algorithm"}


def c3_config(frames: int, chunk: int, world: int) -> dict:
    """The headline workload's config, shared by both arms (the reference arm
    times a bounded sample of it, described in its cpu_baseline.sample)."""
    return {"workload": WORKLOAD, "frames_per_point_per_gpu": frames, "ebno_db": list(EBNO), "chunk": chunk,
            "parallelism": f"frame-sharded x{world}",
            "l2": f"inputs larger than L2 ({frames * N * 4 / 1e6:.0f} MB per point)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle

    threads = oracle.cpu_count()
    fpp = args.cpu_frames or max(2048, 128 * threads)  # ~10 s of oracle work on 16 threads
    vals = []
    for s in range(args.warmup + args.steps):
        v, busy = cpu_hybrid_sample(fpp if s >= args.warmup else max(8, threads), threads)
        if s >= args.warmup:
            vals.append((v, busy))
    value = float(np.mean([v for v, _ in vals]))
    ms = float(np.mean([b for _, b in vals])) * 1e3
    sample = (f"{fpp} frames per Eb/N0 point x {len(EBNO)} points per step (host PCG64 frames, fp64 oracle port on "
              f"{threads} threads; the port is {PORT_OVER_REF:.2f}x the untouched Python reference on the same "
              "frames and cores, profiles/ref_vs_port.json)")
    line = {
        "metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": c3_config(args.frames, args.chunk or args.frames, world),
        "cpu_baseline": {"value": value, "unit": "Gbit/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm --
def run_gpu(args):
    import torch
    import torch.distributed as dist

    torch, dist, rank, world, local = _gpu_common(args)

    from paper_1609_09358_b200 import BpConfig, CodeConfig, HybridDecoder, SclConfig
    from paper_1609_09358_b200 import _native as nat
    from paper_1609_09358_b200.channel import ebno_to_sigma
    from paper_1609_09358_b200.shard import max_over_ranks, shard_range

    lib = nat.load()
    code = CodeConfig(N, K, crc=16)
    m = code.message_len
    B = args.frames
    dev = torch.device("cuda", local)
    dc = nat.device_code(code)
    MW = (m + 31) // 32
    # inputs resident in HBM before timing: per point B frames keyed by the global frame index
    llr = torch.empty((len(EBNO), B, N), dtype=torch.float32, device=dev)
    msg = torch.empty((len(EBNO), B, MW), dtype=torch.int32, device=dev)
    for p, eb in enumerate(EBNO):
        sigma = ebno_to_sigma(eb, code.rate)
        nat.check(lib.pc_gen_frames(SEED, p, shard_range(rank, world, B)[0], B, sigma, dc.ref, msg[p].data_ptr(),
                                    llr[p].data_ptr(),
                                    nat.stream_handle()), "pc_gen_frames")
    dec = HybridDecoder(code, BpConfig(i_max=IMAX), SclConfig(LIST), capacity=B, chunk=args.chunk or B)
    # the paper's Fig. 2 across batches: points alternate between two decoders and
    # run(join=False) lets point p+1's BP stage start beside point p's SCL stage
    # (whose last few frames at a high Eb/N0 leave most SMs idle)
    twin = HybridDecoder(code, BpConfig(i_max=IMAX), SclConfig(LIST), capacity=B, chunk=args.chunk or B)
    decs = (dec, twin)
    errs = torch.zeros((len(EBNO), 2), dtype=torch.int64, device=dev)

    def one_step(overlap):
        for p in range(len(EBNO)):
            if not overlap:
                dec.join_streams()
                twin.join_streams()
            decs[p % 2].run(llr[p], B, join=False)
        for d in decs:
            d.join_streams()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed_steps(overlap):
        """K steps on the device (events on the launching streams, barrier +
        synchronize on both sides); returns (ms, K1 ms, K2+K3 ms, clocks)."""
        for d in decs:
            d.kernel_events = []
            d.scl_events = []
        with ClockSampler(local) as clk:
            barrier()
            t_start = torch.cuda.Event(enable_timing=True)
            t_end = torch.cuda.Event(enable_timing=True)
            t_start.record()
            for _ in range(args.steps):
                one_step(overlap)
            t_end.record()
            barrier()
        k1 = sum(a.elapsed_time(b) for d in decs for a, b in d.kernel_events)
        k3 = sum(a.elapsed_time(b) for d in decs for a, b in d.scl_events)
        for d in decs:
            d.kernel_events = None
            d.scl_events = None
        return t_start.elapsed_time(t_end), k1, k3, clk.summary()

    for _ in range(args.warmup):
        one_step(False)
        one_step(True)
    barrier()

    # ---- timed region: the points one after another (each point's K1 -> K2 -> K3
    # complete before the next point's K1), so K1's events time K1 with the GPU
    # to itself -- the roofline and the shares below come from this region ----
    elapsed_ms, k1_ms, scl_ms, ck = timed_steps(False)
    # ---- second timed region: the paper's Fig. 2 across points -- point p+1's
    # BP stage starts beside point p's SCL tail (two decoders, run(join=False)) --
    ov_ms, ov_k1_ms, _, ov_ck = timed_steps(True)

    lat_p50, gammas, iters_sum, pt_ms = [[] for _ in EBNO], [[] for _ in EBNO], [0] * len(EBNO), [0.0] * len(EBNO)
    # statistics pass (untimed; one point at a time): gamma, iterations,
    # latency, FER and each point's own device time
    for p in range(len(EBNO)):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        dec.run(llr[p], B)
        b.record()
        dec.sync()
        pt_ms[p] = a.elapsed_time(b) * args.steps
        r = dec.host_results()
        gammas[p] = float((~r["converged"]).mean())
        iters_sum[p] = int(r["iters"].astype(np.int64).sum())
        st = r["stamps"]
        c = np.arange(B) // dec.chunk
        done = np.where(r["converged"], r["t_bp"], r["t_scl"])
        lat_p50[p] = float(np.median(done - st[c, 0])) * 1e-6
        nat.check(lib.pc_count_errors(dec.payload.data_ptr(), msg[p].data_ptr(), B, m, errs[p].data_ptr(),
                                      nat.stream_handle()), "pc_count_errors")
    torch.cuda.synchronize()
    latency_ops = latency_operating_points(torch, code, llr, dev) if rank == 0 else None
    # whole-job statistics: exact integer counters summed over the ranks (off
    # the timed path); the roofline below uses this rank's own iterations and
    # its own K1 time
    local_iters = list(iters_sum)
    stats = torch.tensor([[iters_sum[p], round(gammas[p] * B), int(errs[p, 0]), int(errs[p, 1])]
                          for p in range(len(EBNO))], dtype=torch.int64, device=COMM)
    if world > 1:
        dist.all_reduce(stats)
    stats = stats.cpu().numpy()
    errs_h = stats[:, 2:4]
    for p in range(len(EBNO)):
        iters_sum[p] = int(stats[p, 0])
        gammas[p] = float(stats[p, 1]) / (B * world)

    max_ms = max_over_ranks(elapsed_ms, device=COMM)
    bits_step = B * m * len(EBNO)
    value = world * bits_step * args.steps / (max_ms * 1e-3) / 1e9
    ov_max_ms = max_over_ranks(ov_ms, device=COMM)

    # ---- roofline of the dominant kernel (K1): algorithmic exact-g evaluations / K1 time ----
    n = code.n
    g_per_step = sum(local_iters) * 2 * n * N  # iterations are deterministic per input set
    bp_ms_step = k1_ms / args.steps
    roofline = k1_roofline(torch, dev, N, g_per_step, bp_ms_step * 1e-3, ck, dec.chunk)
    roofline["traffic_source"] = "profiles/bp_kernel_ncu.json: dram__bytes_read+write per frame x frames per launch"
    # K1's own HBM traffic: read the LLRs, write payload + iters + flag + stamp per frame
    roofline["hbm_gbs"] = len(EBNO) * B * (4 * N + 4 * MW + 4 + 1 + 8) / (bp_ms_step * 1e-3) / 1e9
    roofline["bp_share_of_step"] = k1_ms / elapsed_ms
    # K3 (SCL on the BP failures): frames/s and share of the step
    k3 = None
    if scl_ms > 0:
        nscl = sum(round(gammas[p] * B * world) for p in range(len(EBNO))) / world
        k3 = {"kernel": f"k_scl3<{LIST}> (CRC-aided SCL, one warp per frame)", "frames_per_step": nscl,
              "mframes_per_s": nscl * args.steps / (scl_ms * 1e-3) / 1e6, "share_of_step": scl_ms / elapsed_ms,
              "note": "K2 + K3 (compaction + list decoding) from their events in the timed region"}
    # the overlapped schedule: K1 now shares SMs with the previous point's K3,
    # so its own events run longer (the step still gets shorter)
    ov_k1 = k1_roofline(torch, dev, N, g_per_step, ov_k1_ms / args.steps * 1e-3, ov_ck, dec.chunk)
    overlapped = {"value": world * bits_step * args.steps / (ov_max_ms * 1e-3) / 1e9, "unit": "Gbit/s",
                  "ms_per_step": ov_max_ms / args.steps, "k1_frac_contended": ov_k1["frac"],
                  "clocks": ov_ck,
                  "note": "same K steps with point p+1's BP stage launched beside point p's SCL stage (two "
                          "decoders, run(join=False): the paper's Fig. 2 across batches); K1's events then "
                          "include time sharing SMs with K3"}

    # ---- e2e: the public host-buffer call, H2D + decode + D2H inside the timed region ----
    e2e_val = None
    if rank == 0 or world > 1:
        host = [torch.empty((B, N), dtype=torch.float32, pin_memory=True) for _ in EBNO]
        for p in range(len(EBNO)):
            host[p].copy_(llr[p])
        torch.cuda.synchronize()
        dec.decode_host_many(host * args.steps)  # warm-up: allocates the double and pinned result buffers
        barrier()
        t0 = time.perf_counter()
        # one stream of host batches (all steps x points): the H2D of batch i+1
        # overlaps the decode of batch i, so only the first copy is exposed
        dec.decode_host_many(host * args.steps)
        barrier()
        e2e_s = time.perf_counter() - t0
        e2e_val = world * bits_step * args.steps / max_over_ranks(e2e_s, device=COMM) / 1e9
    h2d = B * N * 4 * len(EBNO)
    d2h = B * (MW * 4 + 1) * len(EBNO)

    cpu = parity = None
    if rank == 0 and not args.no_cpu:
        import oracle

        threads = oracle.cpu_count()
        fpp = args.cpu_frames or max(2048, 128 * threads)  # ~10 s of oracle work on 16 threads
        keep = {}
        v, busy = cpu_hybrid_sample(fpp, threads, keep)
        parity = parity_sample(torch, dev, keep)
        cpu = {"value": v, "unit": "Gbit/s", "cores": threads, "kind": "port",
               "sample": f"{fpp} frames per Eb/N0 point x {len(EBNO)} points, {busy:.1f} s of CPU wall "
                         f"(fp64 oracle port of the reference algorithm, all host threads)"}

    sweep = []
    for p, eb in enumerate(EBNO):
        ms = pt_ms[p] / args.steps
        sweep.append({"ebno_db": eb, "gbps": B * m / (ms * 1e-3) / 1e9 * world, "ms": ms, "gamma": gammas[p],
                      "mean_bp_iters": iters_sum[p] / (B * world), "p50_latency_ms": lat_p50[p],
                      "fer": float(errs_h[p, 1]) / (B * world), "ber": float(errs_h[p, 0]) / (B * m * world),
                      "frames": B * world, "frame_errors": int(errs_h[p, 1]), "bit_errors": int(errs_h[p, 0]),
                      "frames_to_scl": int(stats[p, 1]), "bp_iterations": int(stats[p, 0])})
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (device Philox-keyed BPSK/AWGN frames, resident in HBM before timing)",
            "config": c3_config(B, dec.chunk, world),
            "p50_latency_ms": float(np.median([s["p50_latency_ms"] for s in sweep])),
            "latency_operating_points": latency_ops,
            "sweep": sweep,
            "roofline": roofline,
            "k3": k3,
            "overlapped": overlapped,
            "cpu_baseline": cpu,
            "parity_sample": parity,
            "e2e": {"value": e2e_val, "unit": "Gbit/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": args.steps * len(EBNO) * ((B + dec.chunk - 1) // dec.chunk) * dec.launches_per_chunk,
            "clocks": ck,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0

def latency_operating_points(torch, code, llr, dev):
    """p50 frame latency under the reference's semantic (a frame's latency runs
    from its BP batch's start to its final decision, hybrid.py:56-66, sim.py:199)
    at small batches: chunks of 32 frames (the reference's bp_batch_size) and
    1024 frames over 4096 frames per point (the chunks' list decoding on up
    to 8 concurrent SCL streams), and one frame alone on the GPU (64
    single-frame runs per point).  Untimed for the headline value."""
    from paper_1609_09358_b200 import BpConfig, HybridDecoder, SclConfig

    out = []
    pts = [p for p, eb in enumerate(EBNO) if eb in (1.0, 2.0, 3.0, 4.0)]
    NF = min(4096, llr.shape[1])
    for ch in (32, 1024):
        d = HybridDecoder(code, BpConfig(i_max=IMAX), SclConfig(LIST), capacity=NF, chunk=ch, device=dev)
        for p in pts:
            d.run(llr[p], NF).sync()  # warm-up
            t0 = time.perf_counter()
            d.run(llr[p], NF).sync()
            wall = time.perf_counter() - t0
            r = d.host_results()
            c = np.arange(NF) // ch
            done = np.where(r["converged"], r["t_bp"], r["t_scl"])
            lat = (done - r["stamps"][c, 0]) * 1e-6
            out.append({"ebno_db": EBNO[p], "chunk": ch, "frames": NF, "p50_ms": float(np.median(lat)),
                        "p99_ms": float(np.percentile(lat, 99)), "gbps_wall": NF * code.message_len / wall / 1e9,
                        "scl_streams": len(d.s_scls)})
    d1 = HybridDecoder(code, BpConfig(i_max=IMAX), SclConfig(LIST), capacity=1, chunk=1, device=dev)
    for p in pts:
        lat = []
        for f in range(65):
            d1.run(llr[p][f:f + 1], 1).sync()
            r = d1.host_results()
            done = r["t_bp"][0] if r["converged"][0] else r["t_scl"][0]
            if f:  # the first run is a warm-up
                lat.append((done - r["stamps"][0, 0]) * 1e-6)
        out.append({"ebno_db": EBNO[p], "chunk": 1, "frames": 64, "p50_ms": float(np.median(lat)),
                    "p99_ms": float(np.percentile(lat, 99)), "note": "one frame alone on the GPU"})
    return out


# ------------------------------------------------------ secondary workloads --
COMM = None  # device of the collective tensors (the GPU under NCCL, the CPU under gloo)


def _gpu_common(args):
    """One process per GPU over NCCL.  When more ranks than GPUs are started
    (a test of the multi-rank path on a smaller box) the ranks share GPUs and
    the collectives run over gloo on CPU tensors."""
    global COMM
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    # NCCL's INIT log (one "Init COMPLETE" per rank) goes to stderr, so the rank
    # count of a run is visible; the JSON line on stdout stays alone
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    ngpu = torch.cuda.device_count()
    local = local % max(1, ngpu)
    torch.cuda.set_device(local)
    COMM = torch.device("cuda", local)
    if world > 1:
        if ngpu >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
            COMM = torch.device("cpu")
    return torch, dist, rank, world, local


def _cpu_sample(sample, fpp, fixed, min_s=2.0, cap=1 << 16):
    """Run sample(fpp) -> (busy_s, bits), growing fpp 4x until the oracle's
    decode takes at least min_s of wall (a bounded but measurable sample)."""
    busy, bits = sample(fpp)
    while not fixed and busy < min_s and fpp < cap:
        fpp = min(cap, fpp * 4)
        busy, bits = sample(fpp)
    return fpp, busy, bits


BP_WORKLOADS = {
    "c1": {"N": 128, "K": 64, "pts": (2.0,), "pid": 30, "B": 1 << 20, "cfg": 0, "fixed_cap": True,
           "metric": "decoded info Gbit/s, inter-frame BP N=128 R=1/2 (i_max=50, CRC stop), Eb/N0 2 dB",
           "workload": "BP-only N=128 K=64 (48 payload + CRC-16) i_max=50 CRC stop (BASELINE configs[0])",
           "kernel": "k_bp2<7,32,0,persistent>"},
    "c4": {"N": 4096, "K": 2048, "pts": (2.0, 3.0), "pid": 10, "B": 1 << 16, "cfg": 3,
           "metric": "decoded info Gbit/s, inter-frame BP N=4096 R=1/2 (i_max=50, CRC stop), Eb/N0 2 and 3 dB",
           "workload": "BP-only N=4096 K=2048 (2032 payload + CRC-16) i_max=50 CRC stop (BASELINE configs[3])",
           "kernel": "k_bp2<12,512,0> (register/shuffle BP, 512 threads/frame)"},
}


def run_bp_workload(args):
    """BASELINE configs[0] (c1: BP N=128 K=64, 2 dB) and configs[3] (c4:
    inter-frame BP N=4096 K=2048, 2 and 3 dB): i_max=50, CRC stop; frames
    sharded across ranks (weak)."""
    import ctypes

    wl = BP_WORKLOADS[args.workload]
    torch, dist, rank, world, local = _gpu_common(args)
    from paper_1609_09358_b200 import BpConfig, CodeConfig
    from paper_1609_09358_b200 import _native as nat
    from paper_1609_09358_b200.channel import ebno_to_sigma
    from paper_1609_09358_b200.shard import max_over_ranks, shard_range

    lib = nat.load()
    n4, k4, pts = wl["N"], wl["K"], wl["pts"]
    code = CodeConfig(n4, k4, crc=16)
    m, MW = code.message_len, (code.message_len + 31) // 32
    B = args.frames if args.frames != (1 << 17) else wl["B"]
    dev = torch.device("cuda", local)
    dc = nat.device_code(code)
    st = nat.stream_handle()
    llr = torch.empty((len(pts), B, n4), dtype=torch.float32, device=dev)
    msg = torch.empty((len(pts), B, MW), dtype=torch.int32, device=dev)
    for p, eb in enumerate(pts):
        nat.check(lib.pc_gen_frames(SEED, wl["pid"] + p, shard_range(rank, world, B)[0], B, ebno_to_sigma(eb, code.rate),
                                    dc.ref, msg[p].data_ptr(), llr[p].data_ptr(), st), "pc_gen_frames")
    pay = torch.empty((B, MW), dtype=torch.int32, device=dev)
    iters = torch.empty((len(pts), B), dtype=torch.int32, device=dev)
    conv = torch.empty((len(pts), B), dtype=torch.uint8, device=dev)
    errs = torch.zeros((len(pts), 2), dtype=torch.int64, device=dev)
    cfg = BpConfig(i_max=IMAX, stop_mode="crc").native()
    work = torch.empty(1, dtype=torch.int32, device=dev)  # frame counter: persistent K1 at small N
    cfg.work = work.data_ptr()

    def step(events=None):
        for p in range(len(pts)):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            nat.check(lib.pc_bp_decode(llr[p].data_ptr(), B, dc.ref, ctypes.byref(cfg), None, pay.data_ptr(), None,
                                       None, iters[p].data_ptr(), conv[p].data_ptr(), None, st), "pc_bp_decode")
            b.record()
            if events is not None:
                events[p].append((a, b))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    events = [[] for _ in pts]
    with ClockSampler(local) as clocks:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            step(events)
        t1.record()
        barrier()
    ms = t0.elapsed_time(t1)
    pt_ms = [sum(a.elapsed_time(b) for a, b in ev) / args.steps for ev in events]
    for p in range(len(pts)):  # FER on the last step's payloads, recomputed per point (untimed)
        nat.check(lib.pc_bp_decode(llr[p].data_ptr(), B, dc.ref, ctypes.byref(cfg), None, pay.data_ptr(), None,
                                   None, iters[p].data_ptr(), conv[p].data_ptr(), None, st), "pc_bp_decode")
        nat.check(lib.pc_count_errors(pay.data_ptr(), msg[p].data_ptr(), B, m, errs[p].data_ptr(), st), "count")
    torch.cuda.synchronize()
    it_local = iters.to(torch.int64).sum(dim=1)
    # exact whole-job counters: iterations, bit errors, frame errors, BP failures summed over ranks
    stats = torch.stack([it_local, errs[:, 0], errs[:, 1], (conv == 0).to(torch.int64).sum(dim=1)], dim=1).to(COMM)
    if world > 1:
        dist.all_reduce(stats)
    stats = stats.cpu().numpy()
    it_sum = it_local.cpu().numpy()  # this rank's, for its own roofline
    max_ms = max_over_ranks(ms, device=COMM)
    value = world * B * m * len(pts) * args.steps / (max_ms * 1e-3) / 1e9
    g_step = int(it_sum.sum()) * 2 * code.n * n4
    # e2e: pinned host LLRs -> device, decode, payload + flags -> host, every step
    host = [torch.empty((B, n4), dtype=torch.float32, pin_memory=True) for _ in pts]
    for p in range(len(pts)):
        host[p].copy_(llr[p])
    pay_h = [torch.empty((B, MW), dtype=torch.int32, pin_memory=True) for _ in pts]
    conv_h = [torch.empty(B, dtype=torch.uint8, pin_memory=True) for _ in pts]
    # e2e units: each point's batch in NC chunks, NBUF chunk buffers, so the
    # first exposed copy is one chunk and the link streams ahead of the decode
    NC = 4 if B % 4 == 0 else 1  # (8 chunks measured slower: launch tails)
    Bc = B // NC
    # a deep ring of device input buffers (up to 6 GB of HBM): the link copies
    # ahead through slow chunks, so it keeps pace where a decode is shorter than its copy
    NBUF = max(2, min(args.steps * len(pts) * NC, 16, int(6e9 // (Bc * n4 * 4))))
    dbufs = [torch.empty((Bc, n4), dtype=torch.float32, device=dev) for _ in range(NBUF)]
    s_copy = torch.cuda.Stream(device=dev)

    def e2e_run(nsteps):
        cur = torch.cuda.current_stream(dev)
        seq = [(p, c) for _ in range(nsteps) for p in range(len(pts)) for c in range(NC)]
        h2d, done = [None] * len(seq), [None] * len(seq)

        def issue(i):
            p, c = seq[i]
            with torch.cuda.stream(s_copy):
                if i >= NBUF:
                    s_copy.wait_event(done[i - NBUF])
                dbufs[i % NBUF].copy_(host[p][c * Bc:(c + 1) * Bc], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_copy)
                h2d[i] = e

        for i in range(min(NBUF - 1, len(seq))):
            issue(i)
        for i, (p, c) in enumerate(seq):
            if i + NBUF - 1 < len(seq):
                issue(i + NBUF - 1)
            cur.wait_event(h2d[i])
            nat.check(lib.pc_bp_decode(dbufs[i % NBUF].data_ptr(), Bc, dc.ref, ctypes.byref(cfg), None,
                                       pay.data_ptr() + 4 * MW * c * Bc, None, None, iters[p].data_ptr() + 4 * c * Bc,
                                       conv[p].data_ptr() + c * Bc, None, st), "pc_bp_decode")
            e = torch.cuda.Event()
            e.record(cur)
            done[i] = e
            if c == NC - 1:  # the point's payloads and flags back to the host
                pay_h[p].copy_(pay, non_blocking=True)
                conv_h[p].copy_(conv[p], non_blocking=True)
        torch.cuda.synchronize()

    fixed = None
    if wl.get("fixed_cap"):
        # BASELINE configs[0]'s fixed iteration cap: stop rule "none", every frame
        # runs exactly i_max iterations (deterministic work for the roofline)
        cfg_none = BpConfig(i_max=IMAX, stop_mode="none").native()
        cfg_none.work = work.data_ptr()

        def step_none():
            nat.check(lib.pc_bp_decode(llr[0].data_ptr(), B, dc.ref, ctypes.byref(cfg_none), None, pay.data_ptr(),
                                       None, None, iters[0].data_ptr(), conv[0].data_ptr(), None, st), "bp none")

        for _ in range(args.warmup):
            step_none()
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            step_none()
        b.record()
        barrier()
        fms = max_over_ranks(a.elapsed_time(b) / args.steps, device=COMM)
        fg = B * IMAX * 2 * code.n * n4 / (fms * 1e-3) / 1e9
        rf = k1_roofline(torch, dev, n4, B * IMAX * 2 * code.n * n4, fms * 1e-3, None)
        fixed = {"stop_mode": "none", "i_max": IMAX, "ms_per_batch": fms,
                 "frame_iterations_per_s": world * B * IMAX / (fms * 1e-3),
                 "gbps": world * B * m / (fms * 1e-3) / 1e9, "achieved_gg_s": fg, "frac": rf["frac"],
                 "frac_alg": rf["frac_alg"]}
    e2e_run(1)
    barrier()
    te = time.perf_counter()
    e2e_run(args.steps)
    barrier()
    e2e_val = world * B * m * len(pts) * args.steps / max_over_ranks(time.perf_counter() - te, device=COMM) / 1e9
    roofline = k1_roofline(torch, dev, n4, g_step, sum(pt_ms) * 1e-3, clocks.summary())
    if rank == 0:
        cpu = None
        if not args.no_cpu:
            import oracle
            from paper_1609_09358_b200.channel import frame_rng, make_frame

            threads = oracle.cpu_count()

            def sample(fpp):
                busy, bits = 0.0, 0
                for p, eb in enumerate(pts):
                    sig = ebno_to_sigma(eb, code.rate)
                    L = np.array([make_frame(code, sig, frame_rng(SEED, wl["pid"] + p, f))[1] for f in range(fpp)])
                    t = time.perf_counter()
                    oracle.bp_batch(L, code, i_max=IMAX, stop_mode="crc", nthreads=threads)
                    busy += time.perf_counter() - t
                    bits += fpp * m
                return busy, bits

            fpp, busy, bits = _cpu_sample(sample, args.cpu_frames or max(32, 2 * threads), bool(args.cpu_frames))
            cpu = {"value": bits / busy / 1e9, "unit": "Gbit/s", "cores": threads, "kind": "port",
                   "sample": f"{fpp} frames per Eb/N0 point x {len(pts)} points, {busy:.1f} s of CPU wall "
                             f"(fp64 oracle port of bp_decode, all host threads)"}
        line = {
            "metric": wl["metric"],
            "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (device Philox-keyed BPSK/AWGN frames, resident in HBM before timing)",
            "config": {"workload": wl["workload"], "frames_per_point_per_gpu": B, "ebno_db": list(pts),
                       "parallelism": f"frame-sharded x{world}",
                       "l2": f"inputs larger than L2 ({B * n4 * 4 / 1e6:.0f} MB per point)"},
            "sweep": [{"ebno_db": eb, "gbps": world * B * m / (pt_ms[p] * 1e-3) / 1e9, "ms": pt_ms[p],
                       "mean_bp_iters": float(stats[p, 0]) / (B * world), "fer": float(stats[p, 2]) / (B * world),
                       "ber": float(stats[p, 1]) / (B * m * world), "frames": B * world,
                       "bp_iterations": int(stats[p, 0]), "bit_errors": int(stats[p, 1]),
                       "frame_errors": int(stats[p, 2]), "bp_failures": int(stats[p, 3])}
                      for p, eb in enumerate(pts)],
            "roofline": roofline,
            "fixed_cap": fixed,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "Gbit/s", "h2d_bytes_per_step": B * n4 * 4 * len(pts),
                    "d2h_bytes_per_step": B * (MW * 4 + 1) * len(pts)},
            "gpu_launches": args.steps * len(pts),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


SCL_WORKLOADS = {
    "c2": {"N": 1024, "K": 512, "rows": [(32, eb, 40 + p) for p, eb in enumerate(EBNO)], "B": 16384,
           "metric": "SCL decoded info Gbit/s, N=1024 R=1/2 L=32, Eb/N0 1-4 dB (sweep aggregate)",
           "workload": "CRC-aided SCL N=1024 K=512 (496 payload + CRC-16) L=32, Eb/N0 1-4 dB step 0.5 "
                       "(BASELINE configs[1]); value = sum of bits / sum of time over the points"},
    "c5": {"N": 2048, "K": 1024, "rows": [(L, 2.0, 20) for L in (1, 2, 4, 8, 16, 32)], "B": 10_000,
           "metric": "SCL decoded info Gbit/s and latency vs list size, N=2048 R=1/2, Eb/N0 2 dB",
           "workload": "CRC-aided SCL N=2048 K=1024 (1008 payload + CRC-16) L=1..32 at 2 dB (BASELINE "
                       "configs[4]); value = the L=32 line"},
}


def run_scl_workload(args):
    """BASELINE configs[1] (c2: SCL N=1024 K=512 L=32 over 1-4 dB) and
    configs[4] (c5: SCL N=2048 K=1024 at 2 dB, L = 1, 2, 4, 8, 16, 32): batch
    throughput (frames/s, Gbit/s), the batch p50 frame latency (reference
    semantic: batch start -> frame decision) and the single-frame latency (one
    frame alone on the GPU) per row."""
    import ctypes

    wl = SCL_WORKLOADS[args.workload]
    torch, dist, rank, world, local = _gpu_common(args)
    from paper_1609_09358_b200 import CodeConfig, SclConfig
    from paper_1609_09358_b200 import _native as nat
    from paper_1609_09358_b200.channel import ebno_to_sigma
    from paper_1609_09358_b200.shard import max_over_ranks, shard_range

    lib = nat.load()
    n5, k5 = wl["N"], wl["K"]
    code = CodeConfig(n5, k5, crc=16)
    m, MW = code.message_len, (code.message_len + 31) // 32
    B = args.frames if args.frames != (1 << 17) else wl["B"]
    dev = torch.device("cuda", local)
    dc = nat.device_code(code)
    st = nat.stream_handle()
    llr = torch.empty((B, n5), dtype=torch.float32, device=dev)
    msg = torch.empty((B, MW), dtype=torch.int32, device=dev)
    pay = torch.empty((B, MW), dtype=torch.int32, device=dev)
    tdone = torch.empty(B, dtype=torch.int64, device=dev)
    t0s = torch.empty(1, dtype=torch.int64, device=dev)
    errs = torch.zeros((len(wl["rows"]), 2), dtype=torch.int64, device=dev)
    rows = []

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    total_ms, total_bits = 0.0, 0
    with ClockSampler(local) as clocks:
        for li, (L, eb, pid) in enumerate(wl["rows"]):
            nat.check(lib.pc_gen_frames(SEED, pid, shard_range(rank, world, B)[0], B, ebno_to_sigma(eb, code.rate),
                                        dc.ref, msg.data_ptr(), llr.data_ptr(), st), "pc_gen_frames")
            cfg = SclConfig(L).native()

            def dec(nf, stamp=False):
                if stamp:
                    nat.check(lib.pc_stamp(t0s.data_ptr(), st), "stamp")
                nat.check(lib.pc_scl_decode(llr.data_ptr(), nf, None, None, dc.ref, ctypes.byref(cfg), None,
                                            pay.data_ptr(), None, None, None, tdone.data_ptr() if stamp else None,
                                            dc.scl_workspace(cfg).data_ptr(), st), "pc_scl_decode")

            for _ in range(args.warmup):
                dec(B)
            barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.steps):
                dec(B)
            b.record()
            barrier()
            ms = max_over_ranks(a.elapsed_time(b) / args.steps, device=COMM)
            total_ms += ms
            total_bits += world * B * m
            dec(B, stamp=True)
            nat.check(lib.pc_count_errors(pay.data_ptr(), msg.data_ptr(), B, m, errs[li].data_ptr(), st), "count")
            torch.cuda.synchronize()
            p50 = float(np.median((tdone - t0s).cpu().numpy())) * 1e-6
            # single-frame latency: one frame alone on the device, CUDA events
            one = []
            for r in range(20):
                a1 = torch.cuda.Event(enable_timing=True)
                b1 = torch.cuda.Event(enable_timing=True)
                a1.record()
                dec(1)
                b1.record()
                torch.cuda.synchronize()
                one.append(a1.elapsed_time(b1))
            e_t = errs[li].to(COMM)
            if world > 1:  # whole-job error counters
                dist.all_reduce(e_t)
            e = e_t.cpu().numpy()
            rows.append({"L": L, "ebno_db": eb, "ms_per_batch": ms, "frames_per_s": world * B / (ms * 1e-3),
                         "gbps": world * B * m / (ms * 1e-3) / 1e9, "batch_p50_latency_ms": p50,
                         "single_frame_latency_ms": float(np.median(one[5:])), "fer": float(e[1]) / (B * world),
                         "ber": float(e[0]) / (B * m * world), "frames": B * world, "frame_errors": int(e[1]),
                         "bit_errors": int(e[0])})
    if rank == 0:
        cpu = None
        if not args.no_cpu:
            import oracle
            from paper_1609_09358_b200.channel import frame_rng, make_frame

            threads = oracle.cpu_count()
            L, eb, pid = wl["rows"][-1]
            sig = ebno_to_sigma(eb, code.rate)

            def sample(fpp):
                Lr = np.array([make_frame(code, sig, frame_rng(SEED, pid, f))[1] for f in range(fpp)])
                t = time.perf_counter()
                oracle.scl_batch(Lr, code, L, nthreads=threads)
                return time.perf_counter() - t, fpp * m

            fpp, busy, _ = _cpu_sample(sample, args.cpu_frames or max(64, 4 * threads), bool(args.cpu_frames))
            cpu = {"value": fpp * m / busy / 1e9, "unit": "Gbit/s", "cores": threads, "kind": "port",
                   "sample": f"{fpp} frames at L={L}, {eb} dB, {busy:.1f} s of CPU wall "
                             "(fp64 oracle port of scl_decode)"}
        value = rows[-1]["gbps"] if args.workload == "c5" else total_bits / (total_ms * 1e-3) / 1e9
        line = {
            "metric": wl["metric"],
            "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (device Philox-keyed BPSK/AWGN frames, resident in HBM before timing)",
            "config": {"workload": wl["workload"], "frames_per_gpu": B, "parallelism": f"frame-sharded x{world}",
                       "l2": f"inputs {B * n5 * 4 / 1e6:.0f} MB, decode time per batch >> L2 refill"},
            "list_sweep" if args.workload == "c5" else "sweep": rows,
            "roofline": None,
            "cpu_baseline": cpu,
            "gpu_launches": args.steps * len(rows),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=1 << 17, help="frames per Eb/N0 point per GPU")
    ap.add_argument("--chunk", type=int, default=0, help="frames per BP/SCL chunk (0 = whole batch)")
    ap.add_argument("--cpu-frames", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="c3", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="c3 = hybrid sweep (headline); c1 = BP N=128; c2 = SCL N=1024 L=32 sweep; "
                         "c4 = BP N=4096; c5 = SCL N=2048 list-size sweep")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload in BP_WORKLOADS:
        return run_bp_workload(args)
    if args.workload in SCL_WORKLOADS:
        return run_scl_workload(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
