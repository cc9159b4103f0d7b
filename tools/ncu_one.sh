#!/bin/bash
# One full ncu capture of the first launch of kernels matching REGEX at the bench batch.
#   gpurun -- 'bash tools/ncu_one.sh TAG REGEX [COUNT] [SKIP]'
TAG=$1; KRE=$2; CNT=${3:-1}; SKIP=${4:-0}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c $CNT -o $OUT/prof_$TAG \
  python bench.py --batch ${BATCH:-1024} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-configs > $OUT/ncu_$TAG.log 2>&1
tail -2 $OUT/ncu_$TAG.log
