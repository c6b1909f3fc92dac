#!/bin/bash
# SCL A/B across alternative builds of libpolarcuda.so (development aid):
#   tools/scl_variant_probe.sh _libvariants/*.so
for lib in "$@"; do
  cp "$lib" paper_1609_09358_b200/libpolarcuda.so
  echo "== $lib"
  timeout 100 python tools/scl_ab.py 1024 512 32 1.5 8192 > /tmp/ab.log 2>&1; grep -E "v3" /tmp/ab.log; grep -c "True, True, True, True" /tmp/ab.log
  timeout 100 python tools/scl_ab.py 2048 1024 32 2.0 4096 > /tmp/ab.log 2>&1; grep -E "v3" /tmp/ab.log; grep -c "True, True, True, True" /tmp/ab.log
  timeout 100 python tools/scl_ab.py 2048 1024 8 2.0 4096 > /tmp/ab.log 2>&1; grep -E "v3" /tmp/ab.log; grep -c "True, True, True, True" /tmp/ab.log
done
