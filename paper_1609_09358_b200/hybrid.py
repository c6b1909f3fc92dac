"""Hybrid BP -> SCL decoding (reference ``hybrid.py``) as a device pipeline.

The reference runs BP per frame in a producer thread and pushes CRC failures
through a bounded ``queue.Queue`` to SCL worker threads (``hybrid.py:153-258``).
Here the same dataflow is three kernels per chunk of frames, on two CUDA
streams so BP of chunk c+1 overlaps SCL of chunk c (the paper's Fig. 2
scheduling):

    stream bp : stamp -> K1 pc_bp_decode(chunk) -> stamp -> event e_c
    stream scl:                          wait e_c -> stamp -> K2 pc_compact -> K3 pc_scl_decode(queue)

Frames are decided either by K1 (CRC verified) or by K3 from the ORIGINAL
channel LLRs; all outputs are written per frame index, so the answer on a
failed frame is exactly the list decoder's.  The device queue of a chunk
holds every failure of that chunk, so nothing is dropped and nothing blocks.
Per-frame completion times come from ``%globaltimer`` inside the kernels.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, replace

import numpy as np

from . import _native as nat
from .bp import BpConfig, bp_decode_batch
from .codes import CodeConfig, extract_message
from .scl import SclConfig, decision_aided_mask, scl_decode_batch

__all__ = [
    "FrameJob",
    "HybridStats",
    "HybridDecoder",
    "hybrid_decode_frame",
    "hybrid_decode_batch",
    "theoretical_throughput",
    "latency_stats",
]


@dataclass
class FrameJob:
    """One frame in the pipeline (reference hybrid.py:41-66)."""

    frame_id: int
    llrs: np.ndarray
    true_message: np.ndarray | None = None
    status: str = "pending"
    provenance: str = ""
    message: np.ndarray | None = None
    t_enqueue: float = np.nan
    t_bp_start: float = np.nan
    t_bp_end: float = np.nan
    t_scl_start: float = np.nan
    t_scl_end: float = np.nan

    @property
    def latency(self) -> float:
        end = self.t_scl_end if self.status == "scl_done" else self.t_bp_end
        return end - self.t_enqueue


@dataclass
class HybridStats:
    """Aggregates of one batch run (reference hybrid.py:69-86) + p50 latency."""

    frames_total: int
    frames_to_scl: int
    gamma_bp_fer: float
    info_bits: int
    t_bp_bps: float
    t_scl_bps: float
    t_hyb_theo_bps: float
    throughput_bps: float
    bp_busy_s: float
    scl_busy_s: float
    wall_s: float
    overhead_s: float
    latency_avg_s: float
    latency_max_s: float
    latency_p50_s: float = math.nan


def theoretical_throughput(t_bp: float, t_scl: float, gamma: float) -> float:
    """Eq. (1): t_bp t_scl / (t_scl + gamma t_bp) (reference hybrid.py:89-101)."""
    if not (t_bp > 0 and t_scl > 0):
        raise ValueError("throughputs must be positive")
    if not 0.0 <= gamma <= 1.0:
        raise ValueError(f"gamma must lie in [0, 1], got {gamma}")
    if gamma == 0.0:
        return float(t_bp)
    return float(t_bp * t_scl / (t_scl + gamma * t_bp))


def latency_stats(jobs: list[FrameJob]) -> dict[str, float]:
    """Mean / worst latency of the pipeline and both stages (reference hybrid.py:104-124)."""
    if not jobs:
        raise ValueError("no jobs to summarize")
    hyb = np.array([j.latency for j in jobs])
    bp = np.array([j.t_bp_end - j.t_bp_start for j in jobs])
    scl = np.array([j.t_scl_end - j.t_scl_start for j in jobs if j.status == "scl_done"])
    nan = float("nan")
    return {
        "hybrid_avg_s": float(hyb.mean()),
        "hybrid_max_s": float(hyb.max()),
        "bp_avg_s": float(bp.mean()),
        "bp_max_s": float(bp.max()),
        "scl_avg_s": float(scl.mean()) if scl.size else nan,
        "scl_max_s": float(scl.max()) if scl.size else nan,
        "hybrid_p50_s": float(np.median(hyb)),
    }


def _payload(u_hat: np.ndarray, code: CodeConfig) -> np.ndarray:
    return extract_message(u_hat, code)[: code.message_len]


def hybrid_decode_frame(llrs, code: CodeConfig, bp_cfg: BpConfig | None = None, scl_cfg: SclConfig | None = None):
    """One frame: BP (CRC stop), SCL from the same LLRs on failure -> (payload, provenance)."""
    if code.crc is None:
        raise ValueError("hybrid decoding needs a CRC to detect draft failures")
    bp_cfg = replace(bp_cfg or BpConfig(), stop_mode="crc")
    scl_cfg = scl_cfg or SclConfig()
    llrs = np.asarray(llrs, dtype=np.float64)
    draft = bp_decode_batch(llrs[None, :], code, bp_cfg)
    if draft.converged[0]:
        return _payload(draft.u_hat[0], code), "bp"
    res = scl_decode_batch(llrs[None, :], code, scl_cfg)
    return _payload(res.u_hat[0], code), "scl"


class HybridDecoder:
    """Device-resident hybrid pipeline over up to ``capacity`` frames per call.

    ``run(llr)`` takes a CUDA float32 tensor ``[B, N]`` already in HBM and
    leaves per-frame results in preallocated device buffers:
    ``payload [cap, ceil(m/32)] int32``, ``converged``, ``iters``, ``t_bp``,
    ``t_scl`` (globaltimer ns) and per-chunk stamps.
    """

    def __init__(self, code: CodeConfig, bp_cfg: BpConfig | None = None, scl_cfg: SclConfig | None = None,
                 capacity: int = 1 << 16, chunk: int | None = None, overlap: bool = True, device=None,
                 scl_streams: int | None = None):
        if code.crc is None:
            raise ValueError("hybrid decoding needs a CRC to detect draft failures")
        torch = nat.require_device()
        self.torch = torch
        self.lib = nat.load()
        self.code = code
        self.bp_cfg = replace(bp_cfg or BpConfig(), stop_mode="crc")
        self.scl_cfg = scl_cfg or SclConfig()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.device = dev
        self.capacity = int(capacity)
        self.chunk = int(chunk or capacity)
        self.overlap = overlap
        da = decision_aided_mask(code, self.scl_cfg.da_threshold) if self.scl_cfg.da_threshold > 0 else None
        self.dc_bp = nat.device_code(code)
        self.dc_scl = nat.device_code(code, da)
        self.nbp = self.bp_cfg.native()
        self.nscl = self.scl_cfg.native()
        cap = self.capacity
        NW = (code.N + 31) // 32
        self.MW = (code.message_len + 31) // 32
        z = dict(device=dev)
        self.payload = torch.zeros((cap, self.MW), dtype=torch.int32, **z)
        self.iters = torch.zeros(cap, dtype=torch.int32, **z)
        self.conv = torch.zeros(cap, dtype=torch.uint8, **z)
        self.t_bp = torch.zeros(cap, dtype=torch.int64, **z)
        self.t_scl = torch.zeros(cap, dtype=torch.int64, **z)
        self.queue = torch.zeros(cap, dtype=torch.int32, **z)
        self.nchunks_max = (cap + self.chunk - 1) // self.chunk
        self.counts = torch.zeros(self.nchunks_max, dtype=torch.int32, **z)
        # stamps per chunk: [start, bp_end, scl_start, scl_end]
        self.stamps = torch.zeros((self.nchunks_max, 4), dtype=torch.int64, **z)
        # SCL streams (the reference's SCL workers, hybrid.py:153-231): chunk c's
        # K2 + K3 run on stream c mod S with that stream's own K3 workspace, so
        # the list decoding of small chunks (bp_batch_size = 32: a few failures,
        # one warp each) overlaps instead of queueing one chunk behind the other
        # (default: one per chunk of a full batch, at most 8; 1 without overlap)
        if scl_streams is None:
            scl_streams = min(8, self.nchunks_max) if overlap else 1
        if scl_streams < 1 or (scl_streams > 1 and not overlap):
            raise ValueError("scl_streams must be >= 1 (and 1 without overlap)")
        self.scl_wss = [self.dc_scl.new_scl_workspace(self.nscl) for _ in range(scl_streams)]
        self.scl_ws = self.scl_wss[0]
        self.bp_work = torch.empty(1, dtype=torch.int32, **z)
        self.nbp.work = self.bp_work.data_ptr()
        self.s_bp = torch.cuda.Stream(device=dev)
        # The list decoder's persistent warps get the higher stream priority, so
        # they take SM slots as soon as K1 CTAs (one frame each) retire and the
        # two kernels share the GPU instead of running back to back.
        self.s_scls = ([torch.cuda.Stream(device=dev, priority=-1) for _ in range(scl_streams)] if overlap
                       else [self.s_bp])
        self.s_scl = self.s_scls[0]  # joins the others at the end of run()
        self.kernel_events = None  # set to [] to time every K1 launch with CUDA events on the BP stream
        self.scl_events = None  # set to [] to time every K2 + K3 pair with CUDA events on the SCL stream
        self.launches_per_chunk = 7  # 4 stamp kernels + K1 + K2 + K3 (memset nodes not counted)
        self._llr_dev = None

    def decode_host(self, llr_host, B: int | None = None):
        """End-to-end call with HOST buffers: pinned LLRs [B, N] float32 in,
        payload words [B, ceil(m/32)] (numpy uint32 view) out.  The H2D copy,
        the pipeline and the D2H copy are ordered on the current stream."""
        torch = self.torch
        B = int(llr_host.shape[0] if B is None else B)
        if self._llr_dev is None or self._llr_dev.shape[0] < B:
            self._llr_dev = torch.empty((self.capacity, self.code.N), dtype=torch.float32, device=self.device)
        dst = self._llr_dev[:B]
        dst.copy_(llr_host[:B], non_blocking=True)
        self.run(dst, B)
        if getattr(self, "_pay_host", None) is None or self._pay_host.shape[0] < self.capacity:
            self._pay_host = torch.empty((self.capacity, self.MW), dtype=torch.int32, pin_memory=True)
            self._conv_host = torch.empty(self.capacity, dtype=torch.uint8, pin_memory=True)
        self._pay_host[:B].copy_(self.payload[:B], non_blocking=True)
        self._conv_host[:B].copy_(self.conv[:B], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return self._pay_host[:B].numpy().view(np.uint32), self._conv_host[:B].numpy().astype(bool)

    def decode_host_many(self, batches, input_bytes: float = 6e9):
        """End-to-end call over several HOST batches (pinned float32 [B_i, N]):
        the H2D copies of the next batches run on a copy stream while batch i
        decodes (a ring of device input buffers, as many as ``input_bytes`` of
        HBM holds, at least 3), and each batch's payload words and converged
        flags are read back on a second copy stream (PCIe is full duplex) while
        the next batch decodes.  A deep ring lets the link copy ahead through
        the slow points of a sweep, so it keeps pace where a fast point's decode
        is shorter than its copy.  Returns a list of
        (payload words uint32 [B_i, ceil(m/32)], converged bool [B_i]) numpy
        arrays, in order: views of pinned buffers that the next call reuses (copy
        them to keep them).  Results equal ``decode_host`` per batch."""
        torch = self.torch
        dev = self.device
        if not batches:
            return []
        for b in batches:
            if b.shape[0] > self.capacity:
                raise ValueError(f"batch of {b.shape[0]} frames exceeds capacity {self.capacity}")
        N = self.code.N
        # NBUF device input buffers: the copy of batch i+NBUF-1 starts while
        # batch i decodes, so the link keeps copying through short decodes
        # (a fast point's decode can be shorter than its PCIe copy).
        NBUF = max(3, min(len(batches), 16, int(input_bytes // (self.capacity * N * 4))))
        if (getattr(self, "_dbuf", None) is None or self._dbuf[0].shape[0] < self.capacity
                or len(self._dbuf) < NBUF):
            self._dbuf = [torch.empty((self.capacity, N), dtype=torch.float32, device=dev) for _ in range(NBUF)]
            self._s_copy = torch.cuda.Stream(device=dev)
            self._s_back = torch.cuda.Stream(device=dev)
        NBUF = len(self._dbuf)
        cur = torch.cuda.current_stream(dev)
        outs = []
        h2d = [None] * len(batches)
        done = [None] * len(batches)

        def issue_h2d(i):
            buf = self._dbuf[i % NBUF]
            with torch.cuda.stream(self._s_copy):
                if i >= NBUF:  # the buffer is free once batch i-NBUF has decoded
                    self._s_copy.wait_event(done[i - NBUF])
                buf[: batches[i].shape[0]].copy_(batches[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self._s_copy)
            h2d[i] = ev

        # Batches alternate between this decoder and a twin (same code and
        # configuration, own result buffers), so the D2H copy of batch i runs on
        # the copy stream while batch i+1 decodes.
        if getattr(self, "_twin", None) is None:
            self._twin = HybridDecoder(self.code, self.bp_cfg, self.scl_cfg, capacity=self.capacity,
                                       chunk=self.chunk, overlap=self.overlap, device=self.device,
                                       scl_streams=len(self.s_scls))
        decs = (self, self._twin)
        d2h = [None] * len(batches)
        for i in range(min(NBUF - 1, len(batches))):
            issue_h2d(i)
        for i, b in enumerate(batches):
            if i + NBUF - 1 < len(batches):
                issue_h2d(i + NBUF - 1)  # its buffer held batch i-1, decoded already (in stream order)
            B = int(b.shape[0])
            dec = decs[i % 2]
            cur.wait_event(h2d[i])
            if i >= 2:  # batch i-2's results (same decoder) have been copied out
                cur.wait_event(d2h[i - 2])
            # (join=False: batch i+1, on the twin, starts its BP stage beside this SCL stage)
            dec.run(self._dbuf[i % NBUF][:B], B, join=False)
            ev = torch.cuda.Event()
            ev.record(dec.s_scl)  # the SCL stage ends after the batch's last BP launch
            done[i] = ev
            pay, conv = self._pinned_out(i, B)
            with torch.cuda.stream(self._s_back):
                self._s_back.wait_event(ev)
                pay.copy_(dec.payload[:B], non_blocking=True)
                conv.copy_(dec.conv[:B], non_blocking=True)
                e2 = torch.cuda.Event()
                e2.record(self._s_back)
            d2h[i] = e2
            outs.append((pay, conv))
        self._s_copy.synchronize()
        self._s_back.synchronize()
        for d in decs:
            d.join_streams()
        cur.synchronize()
        return [(p.numpy().view(np.uint32), c.numpy().view(np.bool_)) for p, c in outs]

    def _pinned_out(self, i: int, B: int):
        """Pinned host result buffers for batch slot i (allocated once; pinning is slow)."""
        torch = self.torch
        pool = getattr(self, "_pin_pool", None)
        if pool is None:
            pool = self._pin_pool = []
        while len(pool) <= i:
            pool.append((torch.empty((self.capacity, self.MW), dtype=torch.int32, pin_memory=True),
                         torch.empty(self.capacity, dtype=torch.uint8, pin_memory=True)))
        pay, conv = pool[i]
        return pay[:B], conv[:B]

    def _st(self, s) -> int:
        return int(s.cuda_stream)

    def run(self, llr, B: int | None = None, join: bool = True, graph: bool = False):
        """Enqueue the pipeline for ``llr[:B]`` (CUDA float32).  Returns immediately;
        call ``sync()`` (or read results) afterwards.

        ``join=False`` leaves the BP and SCL streams running after the call
        (the caller's current stream does not wait for them): a second decoder's
        batch can then start its BP stage while this batch is still in its SCL
        stage (the paper's Fig. 2 overlap across batches).  This decoder's own
        next batch still starts its BP stage only after this batch's SCL stage
        (its buffers are reused); call ``join_streams()`` before reading results.

        ``graph=True`` replays a CUDA graph of the whole pipeline (every chunk's
        stamps, K1, K2 and K3 on their streams) captured on the first call for
        this input buffer and batch size: one launch instead of seven per
        chunk from Python, for loops over small chunks that reuse one input
        buffer.  The first call runs eagerly and captures; the graph's work is
        ordered on the caller's stream (``join`` is implied)."""
        if graph:
            return self._run_graph(llr, B)
        torch = self.torch
        N = self.code.N
        if not (hasattr(llr, "is_cuda") and llr.is_cuda):
            raise ValueError("HybridDecoder.run takes a CUDA tensor (use decode_host for host buffers)")
        if llr.dtype != torch.float32 or llr.dim() != 2 or llr.shape[1] != N:
            raise ValueError(f"expected float32 llrs of shape (B, {N}), got {llr.dtype} {tuple(llr.shape)}")
        if llr.device != self.device:
            raise ValueError(f"llrs are on {llr.device}, the decoder on {self.device}")
        if not llr.is_contiguous() or llr.data_ptr() % 16:
            raise ValueError("llrs must be contiguous and 16-byte aligned (TMA row copies)")
        B = int(llr.shape[0] if B is None else B)
        if B > llr.shape[0] or B < 0:
            raise ValueError(f"B={B} outside the {llr.shape[0]} rows of llrs")
        if B > self.capacity:
            raise ValueError(f"batch of {B} frames exceeds capacity {self.capacity}")
        lib, chk = self.lib, nat.check
        cur = torch.cuda.current_stream(self.device)
        self.s_bp.wait_stream(cur)
        for s_ in self.s_scls:
            s_.wait_stream(cur)
        # this decoder's buffers (payload, flags, queue) are reused: the BP stage of
        # this batch waits for the previous batch's SCL stage when it was not joined
        # (s_scl has joined the other SCL streams at the end of the previous run)
        self.s_bp.wait_stream(self.s_scl)
        bp_ref, scl_ref = ctypes.byref(self.nbp), ctypes.byref(self.nscl)
        base_llr = llr.data_ptr()
        self._events = []
        nss = len(self.s_scls)
        for c, b0 in enumerate(range(0, B, self.chunk)):
            nb = min(self.chunk, B - b0)
            s_scl = self.s_scls[c % nss]
            sb, ss = self._st(self.s_bp), self._st(s_scl)
            st = self.stamps[c]
            chk(lib.pc_stamp(st.data_ptr(), sb), "pc_stamp")
            if self.kernel_events is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(self.s_bp)
            chk(
                lib.pc_bp_decode(
                    base_llr + 4 * N * b0, nb, self.dc_bp.ref, bp_ref, None,
                    self.payload.data_ptr() + 4 * self.MW * b0, None, None,
                    self.iters.data_ptr() + 4 * b0, self.conv.data_ptr() + b0, self.t_bp.data_ptr() + 8 * b0, sb,
                ),
                "pc_bp_decode",
            )
            if self.kernel_events is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(self.s_bp)
                self.kernel_events.append((e0, e1))
            chk(lib.pc_stamp(st.data_ptr() + 8, sb), "pc_stamp")
            if self.overlap:
                ev = torch.cuda.Event()
                ev.record(self.s_bp)
                s_scl.wait_event(ev)
                self._events.append(ev)
            chk(lib.pc_stamp(st.data_ptr() + 16, ss), "pc_stamp")
            if self.scl_events is not None:
                e2 = torch.cuda.Event(enable_timing=True)
                e2.record(s_scl)
            q = self.queue.data_ptr() + 4 * b0
            cnt = self.counts.data_ptr() + 4 * c
            chk(lib.pc_compact(self.conv.data_ptr() + b0, nb, q, cnt, None, ss), "pc_compact")
            chk(
                lib.pc_scl_decode(
                    base_llr + 4 * N * b0, nb, q, cnt, self.dc_scl.ref, scl_ref, None,
                    self.payload.data_ptr() + 4 * self.MW * b0, None, None, None,
                    self.t_scl.data_ptr() + 8 * b0, self.scl_wss[c % nss].data_ptr(), ss,
                ),
                "pc_scl_decode",
            )
            if self.scl_events is not None:
                e3 = torch.cuda.Event(enable_timing=True)
                e3.record(s_scl)
                self.scl_events.append((e2, e3))
            chk(lib.pc_stamp(st.data_ptr() + 24, ss), "pc_stamp")
        for s_ in self.s_scls[1:]:
            self.s_scl.wait_stream(s_)
        self._B = B
        if join:
            self.join_streams()
        return self

    def _run_graph(self, llr, B):
        torch = self.torch
        if self.kernel_events is not None or self.scl_events is not None:
            raise ValueError("graph=True does not record per-kernel timing events")
        B = int(llr.shape[0] if B is None else B)
        key = (llr.data_ptr(), B, tuple(llr.shape))
        graphs = getattr(self, "_graphs", None)
        if graphs is None:
            graphs = self._graphs = {}
        g = graphs.get(key)
        if g is None:
            self.run(llr, B)  # eager (validates, loads modules, first results)
            cur = torch.cuda.current_stream(self.device)
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(cur)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self.run(llr, B)  # enqueued on the BP / SCL streams, which join the capture
            cur.wait_stream(side)
            if len(graphs) >= 8:  # a bounded cache: drop the oldest capture
                graphs.pop(next(iter(graphs)))
            graphs[key] = g
            return self
        g.replay()
        self._B = B
        return self

    def join_streams(self):
        """The caller's current stream waits for this decoder's BP and SCL stages."""
        cur = self.torch.cuda.current_stream(self.device)
        cur.wait_stream(self.s_bp)
        cur.wait_stream(self.s_scl)
        return self

    def sync(self):
        self.torch.cuda.current_stream(self.device).synchronize()
        return self

    def warm(self):
        """One all-zero frame through the pipeline (K1, K2 and K3 are all
        launched; K3 reads its frame count on the device): the one-time costs
        of a decoder -- lazy loading of its
        kernels' modules, first-launch attribute calls, the caching allocator --
        are paid here, not by the first batch a caller times."""
        torch = self.torch
        z = torch.zeros((1, self.code.N), dtype=torch.float32, device=self.device)
        self.run(z, 1).sync()

    def host_results(self):
        """Copy per-frame results of the last run to numpy (after sync)."""
        B = self._B
        nch = (B + self.chunk - 1) // self.chunk
        return dict(
            payload=self.payload[:B].cpu().numpy().view(np.uint32),
            converged=self.conv[:B].cpu().numpy().astype(bool),
            iters=self.iters[:B].cpu().numpy(),
            t_bp=self.t_bp[:B].cpu().numpy(),
            t_scl=self.t_scl[:B].cpu().numpy(),
            stamps=self.stamps[:nch].cpu().numpy(),
            counts=self.counts[:nch].cpu().numpy(),
        )


def _busy(start, end) -> float:
    """Seconds covered by the union of the [start, end) globaltimer intervals (ns):
    the service time of a stage whose chunks may run concurrently (several SCL
    streams); equal to the sum of the intervals when they do not overlap."""
    iv = sorted(zip((int(a) for a in start), (int(b) for b in end)))
    tot, cur_a, cur_b = 0, None, None
    for a, b in iv:
        if cur_b is None or a > cur_b:
            if cur_b is not None:
                tot += cur_b - cur_a
            cur_a, cur_b = a, b
        else:
            cur_b = max(cur_b, b)
    if cur_b is not None:
        tot += cur_b - cur_a
    return tot * 1e-9


def hybrid_decode_batch(
    jobs: list[FrameJob],
    code: CodeConfig,
    bp_cfg: BpConfig | None = None,
    scl_cfg: SclConfig | None = None,
    *,
    bp_batch_size: int = 32,
    n_scl_workers: int = 2,
    buffer_capacity: int | None = None,
    decoder: "HybridDecoder | None" = None,
) -> HybridStats:
    """Decode jobs through the device pipeline; jobs are completed in place.

    ``bp_batch_size`` is the chunk that shares one BP service interval, as in
    the reference; ``n_scl_workers`` is the number of SCL streams (at most 8):
    the list decoding of that many chunks runs concurrently, as the
    reference's SCL worker threads do; ``buffer_capacity`` is validated for
    API compatibility (the device queue of a chunk always holds all of its
    failures, so it can neither drop nor block).  ``decoder`` reuses a
    ``HybridDecoder`` of the same code across calls (a sweep point's chunks);
    its capacity must hold the jobs and its chunk must equal ``bp_batch_size``.
    """
    if not jobs:
        raise ValueError("no jobs to decode")
    if code.crc is None:
        raise ValueError("hybrid decoding needs a CRC to detect draft failures")
    if bp_batch_size < 1 or n_scl_workers < 1:
        raise ValueError("batch size and worker count must be at least 1")
    if buffer_capacity is not None and buffer_capacity < 1:
        raise ValueError("buffer capacity must be at least 1")
    torch = nat.require_device()
    B = len(jobs)
    llr_host = np.stack([np.asarray(j.llrs, dtype=np.float64) for j in jobs])
    if llr_host.shape[1] != code.N:
        raise ValueError(f"expected {code.N} channel LLRs per job, got {llr_host.shape[1]}")
    if decoder is None:
        # the reference's SCL workers map to SCL streams (concurrent K3 launches)
        dec = HybridDecoder(code, bp_cfg, scl_cfg, capacity=B, chunk=bp_batch_size,
                            scl_streams=min(n_scl_workers, 8, (B + bp_batch_size - 1) // bp_batch_size))
        dec.warm()
    else:
        dec = decoder
        if dec.code is not code or dec.capacity < B or dec.chunk != bp_batch_size:
            raise ValueError("decoder does not match the code, the batch size or the job count")
        if bp_cfg is not None and replace(bp_cfg, stop_mode="crc") != dec.bp_cfg:
            raise ValueError("decoder was built for another BP configuration")
        if scl_cfg is not None and scl_cfg != dec.scl_cfg:
            raise ValueError("decoder was built for another SCL configuration")
    pinned = torch.from_numpy(llr_host.astype(np.float32)).pin_memory()
    t_host0 = time.perf_counter()
    g0 = torch.zeros(1, dtype=torch.int64, device=dec.device)
    nat.check(nat.load().pc_stamp(g0.data_ptr(), nat.stream_handle()), "pc_stamp")
    llr_dev = pinned.to(dec.device, non_blocking=True)
    dec.run(llr_dev).sync()
    r = dec.host_results()
    wall = time.perf_counter() - t_host0
    gbase = int(g0.item())

    def h(g):
        return t_host0 + (np.asarray(g, dtype=np.float64) - gbase) * 1e-9

    m = code.message_len
    bits = nat.unpack_bits(r["payload"], m)
    st = r["stamps"]
    bp_busy = _busy(st[:, 0], st[:, 1])
    scl_busy = _busy(st[:, 2], st[:, 3])  # the SCL streams' union: time any of them is busy
    for b, job in enumerate(jobs):
        c = b // bp_batch_size
        job.t_enqueue = job.t_bp_start = float(h(st[c, 0]))
        job.t_bp_end = float(h(st[c, 1]))
        job.message = bits[b].copy()
        if r["converged"][b]:
            job.status, job.provenance = "bp_done_ok", "bp"
        else:
            job.status, job.provenance = "scl_done", "scl"
            job.t_scl_start = float(h(st[c, 2]))
            job.t_scl_end = max(float(h(r["t_scl"][b])), job.t_scl_start)
    frames_to_scl = int((~r["converged"]).sum())
    gamma = frames_to_scl / B
    bits_total = B * m
    t_bp = bits_total / bp_busy if bp_busy > 0 else math.inf
    t_scl = frames_to_scl * m / scl_busy if frames_to_scl and scl_busy > 0 else math.nan
    theo = t_bp if frames_to_scl == 0 else theoretical_throughput(t_bp, t_scl, gamma)
    lat = latency_stats(jobs)
    return HybridStats(
        frames_total=B,
        frames_to_scl=frames_to_scl,
        gamma_bp_fer=gamma,
        info_bits=bits_total,
        t_bp_bps=t_bp,
        t_scl_bps=t_scl,
        t_hyb_theo_bps=theo,
        throughput_bps=bits_total / wall,
        bp_busy_s=bp_busy,
        scl_busy_s=scl_busy,
        wall_s=wall,
        overhead_s=wall - bp_busy - scl_busy,
        latency_avg_s=lat["hybrid_avg_s"],
        latency_max_s=lat["hybrid_max_s"],
        latency_p50_s=lat["hybrid_p50_s"],
    )
