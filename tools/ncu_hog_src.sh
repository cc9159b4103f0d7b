#!/bin/bash
# ncu --set full of one gradHist launch at the bench batch plus its per-SASS source page
# (stall samples per instruction), for the kernel selected by BL_HOG (v2 default, v3 ...).
#   gpurun -- 'bash tools/ncu_hog_src.sh TAG [v2 v3 ...]'
TAG=${1:-hog}; shift; VERS=${@:-v2}
OUT=gpurun_out; mkdir -p $OUT
for v in $VERS; do
  BL_HOG=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hog" -c 1 -o $OUT/prof_${TAG}_$v \
    python bench.py --batch 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-configs > $OUT/ncu_${TAG}_$v.log 2>&1
  tail -1 $OUT/ncu_${TAG}_$v.log
  ncu -i $OUT/prof_${TAG}_$v.ncu-rep --page source --csv --print-source sass > $OUT/src_${TAG}_$v.csv 2>/dev/null
done
