#!/bin/bash
# Warm C1 / C2 per-kernel times (tools/c1_kernels.sh) for the main build and every variant.
echo "== main"; bash tools/c1_kernels.sh 2>&1 | grep -E "${KRE:-rescore|nms|ert|hog3|sum}"
for v in $(ls -d variants/*/ 2>/dev/null); do n=$(basename $v); echo "== $n"; BL_LIBRARY=$PWD/$v/libblinkline_b200.so bash tools/c1_kernels.sh 2>&1 | grep -E "${KRE:-rescore|nms|ert|hog3|sum}"; done
