#!/bin/bash
# ncu --set full of the gradHist kernel, round-1 (v1) and current (v2), at the bench batch.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-hogab}
for v in ${VERS:-v1 v2}; do
  BL_HOG=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hog" -c 1 -o $OUT/prof_${TAG}_$v \
    python bench.py --batch 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-configs > $OUT/ncu_${TAG}_$v.log 2>&1
  tail -1 $OUT/ncu_${TAG}_$v.log
done
