set -x
timeout 600 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest2.log 2>&1
timeout 300 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 1 --warmup 1 --frames 16384 --no-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_bp_decode -c 1 -o gpurun_out/bp2 -f python tools/profile_kernels.py 16384 1024 > gpurun_out/ncu_bp2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scl -c 1 -o gpurun_out/scl2 -f python tools/profile_kernels.py 1024 2048 > gpurun_out/ncu_scl2.log 2>&1
tail -3 gpurun_out/pytest2.log
