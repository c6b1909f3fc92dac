timeout 900 python -m pytest tests/test_gpu_sim.py -q -rf --timeout 600 > gpurun_out/pytest8.log 2>&1
tail -30 gpurun_out/pytest8.log
