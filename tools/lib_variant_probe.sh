#!/bin/bash
# Time K1 with alternative builds of libpolarcuda.so (development aid):
#   tools/lib_variant_probe.sh _libvariants/*.so
for lib in "$@"; do
  cp "$lib" paper_1609_09358_b200/libpolarcuda.so
  echo "== $lib"
  timeout 200 python tools/bp_tpf_probe.py 1024 2.0 131072 256
  timeout 200 python tools/bp_tpf_probe.py 4096 2.0 32768 512
done
