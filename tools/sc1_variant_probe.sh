#!/bin/bash
# SC kernel variants (development aid): tools/sc1_variant_probe.sh build/variants/*.so
for lib in "$@"; do
  cp "$lib" paper_1609_09358_b200/libpolarcuda.so
  echo "== $lib"
  timeout 300 python tools/sc1_ab.py 2>&1 | grep "ALL_\|L=1 kernel=3\|L=2 kernel"
done
