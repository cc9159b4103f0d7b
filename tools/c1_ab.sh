#!/bin/bash
# C1 / C2 probe of the main build and every variants/*/ build.
echo "== main"; bash tools/c1_probe.sh 2>&1 | head -4
for v in $(ls -d variants/*/ 2>/dev/null); do n=$(basename $v); echo "== $n"; BL_LIBRARY=$PWD/$v/libblinkline_b200.so bash tools/c1_probe.sh 2>&1 | head -4; done
