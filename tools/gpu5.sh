timeout 400 python tools/probe.py 131072 hyb > gpurun_out/probe5.log 2>&1
tail -30 gpurun_out/probe5.log
