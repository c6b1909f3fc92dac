"""Reference acceptance test 08's configuration (N=1024 L=8, 768 frames in
batches of 32) in a fresh process: the Eq. (1) gap of the first call (cold:
lazy kernel loading, allocations) and of repeated calls.
    python tools/eq1_cold_probe.py"""
import sys

sys.path.insert(0, ".")
from paper_1609_09358_b200 import BpConfig, CodeConfig, FrameJob, SclConfig, hybrid_decode_batch  # noqa: E402
from paper_1609_09358_b200.channel import ebno_to_sigma, frame_rng, make_frame  # noqa: E402

code = CodeConfig(1024, 512, crc=16)
for rep in range(3):
    for point, eb in enumerate((1.5, 2.0, 2.5)):
        sigma = ebno_to_sigma(eb, code.rate)
        jobs = []
        for f in range(768):
            m, llr = make_frame(code, sigma, frame_rng(800_000 + point, point, f))
            jobs.append(FrameJob(frame_id=f, llrs=llr, true_message=m))
        st = hybrid_decode_batch(jobs, code, BpConfig(i_max=50), SclConfig(8), bp_batch_size=32, n_scl_workers=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
        gap = abs(st.t_hyb_theo_bps - st.throughput_bps) / st.t_hyb_theo_bps
        print(f"rep {rep} {eb} dB gamma={st.gamma_bp_fer:.3f} model={st.t_hyb_theo_bps / 1e6:.1f} Mbps "
              f"measured={st.throughput_bps / 1e6:.1f} Mbps gap={100 * gap:.1f}%", flush=True)
