PC_SCL_NV=${NV:-4} timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scl -c 1 -o gpurun_out/scl4 -f python tools/profile_kernels.py 1024 4096 > gpurun_out/ncu_scl4.log 2>&1
ls -la gpurun_out/
tail -2 gpurun_out/ncu_scl4.log
