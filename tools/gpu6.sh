timeout 400 python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches6.csv python bench.py --steps 1 --warmup 1 --frames 16384 --no-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_bp2 -c 1 -o gpurun_out/bp6 -f python tools/profile_kernels.py 16384 256 > gpurun_out/ncu_bp6.log 2>&1
tail -c 600 gpurun_out/bench6.json
