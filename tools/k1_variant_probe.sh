#!/bin/bash
# K1 time per launch for alternative builds of libpolarcuda.so (development aid):
#   tools/k1_variant_probe.sh _libvariants/*.so
for lib in "$@"; do
  cp "$lib" paper_1609_09358_b200/libpolarcuda.so
  echo "== $lib"
  for n in 128 1024 4096; do
    timeout 200 python tools/bp_gmode_probe.py $n 2.0 $((131072 * 1024 / n)) 0 0 | cut -c1-120
  done
done
