"""Eq. (1) throughput model (hybrid.theoretical_throughput) vs the measured
hybrid_decode_batch throughput on the device pipeline (reference acceptance
test 08, test_acceptance.py:258-284, for its CPU pipeline).

    python tools/eq1_probe.py
"""
import sys; sys.path.insert(0,'.')
from paper_1609_09358_b200 import BpConfig, CodeConfig, SclConfig, FrameJob, hybrid_decode_batch
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame
code = CodeConfig(1024, 512, crc=16)
for frames, bb in ((768, 32), (8192, 512), (32768, 4096)):
    for eb in (1.5, 2.0, 2.5):
        sigma = ebno_to_sigma(eb, code.rate)
        jobs = []
        for f in range(frames):
            m, l = make_frame(code, sigma, frame_rng(800, 0, f))
            jobs.append(FrameJob(frame_id=f, llrs=l, true_message=m))
        # warm-up at the full size (allocations of this capacity happen once)
        hybrid_decode_batch(jobs, code, BpConfig(i_max=50), SclConfig(8), bp_batch_size=bb)
        st = hybrid_decode_batch(jobs, code, BpConfig(i_max=50), SclConfig(8), bp_batch_size=bb)
        gap = abs(st.t_hyb_theo_bps - st.throughput_bps) / st.t_hyb_theo_bps
        print(frames, bb, eb, f"gamma={st.gamma_bp_fer:.3f} model={st.t_hyb_theo_bps:.3e} measured={st.throughput_bps:.3e} gap={gap*100:.1f}% wall={st.wall_s*1e3:.1f}ms busy={ (st.bp_busy_s+st.scl_busy_s)*1e3:.2f}ms", flush=True)
