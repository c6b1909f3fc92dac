#!/bin/bash
# K1 at N = 128 for alternative builds of libpolarcuda.so (development aid):
#   tools/k1_n128_probe.sh _libvariants/*.so
for lib in "$@"; do
  cp "$lib" paper_1609_09358_b200/libpolarcuda.so
  echo "== $lib"
  timeout 200 python tools/bp_gmode_probe.py 128 2.0 1048576 0 0 | cut -c1-120
done
