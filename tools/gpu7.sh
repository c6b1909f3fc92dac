timeout 900 python tools/fer_parity.py --frames 4000 --device-frames 262144 --out gpurun_out/fer_parity.json > gpurun_out/fer7.log 2>&1
tail -4 gpurun_out/fer7.log
