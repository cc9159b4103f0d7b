#!/bin/bash
# C1 / C2 probe (twice each) of the main build and every variants/*/ build
for v in main $(ls variants 2>/dev/null); do
  L=; [ $v != main ] && L=$PWD/variants/$v/libblinkline_b200.so
  for i in 1 2; do echo "== $v"; BL_LIBRARY=$L bash tools/c1_probe.sh 2>&1 | grep -E "C1 lat|^C2"; done
done
