#!/bin/bash
# One `ncu --set full` capture of the first launch of each named kernel (GPU box, 1 GPU).
#   gpurun -- 'bash tools/ncu_kernels.sh TAG "k_gradhist|k_screen" 2 [bench args]'
TAG=$1; KRE=$2; CNT=${3:-2}; shift 3
ARGS=${@:-"--batch 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c $CNT -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
