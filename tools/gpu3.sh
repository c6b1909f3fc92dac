timeout 600 python -m pytest tests -m gpu -q -rf --timeout 300 -x > gpurun_out/pytest3.log 2>&1
timeout 400 python tools/probe.py 65536 ${PROBE_SECTIONS:-scl,hyb} > gpurun_out/probe3.log 2>&1
tail -3 gpurun_out/pytest3.log
