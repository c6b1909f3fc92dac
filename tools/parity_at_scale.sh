#!/bin/bash
# Parity at scale on the B200 (run under gpurun): SCL C2 (10^5 frames per point)
# and C5, and the randomized sweep (10 seeds x 440 cases).  Outputs in gpurun_out/.
TAG=${1:-r02}
timeout 2400 python tests/parity/scl_parity.py --frames 100000 --out gpurun_out/${TAG}_scl_parity_c2.json > gpurun_out/${TAG}_scl_parity_c2.log 2>&1
timeout 1200 python tests/parity/scl_parity.py --c5 --frames 10000 --out gpurun_out/${TAG}_scl_parity_c5.json > gpurun_out/${TAG}_scl_parity_c5.log 2>&1
for s in 1 2 3 4 5 6 7 8 9 10; do
  timeout 900 python tests/parity/fuzz_parity.py 440 $s > gpurun_out/${TAG}_fuzz_$s.log 2>&1
  tail -1 gpurun_out/${TAG}_fuzz_$s.log
done
tail -n 3 gpurun_out/${TAG}_scl_parity_c2.log gpurun_out/${TAG}_scl_parity_c5.log
