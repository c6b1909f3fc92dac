timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scl -c 1 -o gpurun_out/scl4 -f python tools/profile_kernels.py 1024 4096 > gpurun_out/ncu_scl4.log 2>&1
tail -2 gpurun_out/ncu_scl4.log
