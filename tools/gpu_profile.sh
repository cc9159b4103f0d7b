#!/bin/bash
# Run on the GPU box (via gpurun): parity tests, the bench (ours + reference arm), the ncu
# launch list and one `--set full` capture of the hot kernels.  Outputs land in gpurun_out/.
#   gpurun -- 'bash tools/gpu_profile.sh TAG [KERNEL_REGEX] [COUNT]'
set -u
TAG=${1:-r1}
KRE=${2:-"k_gradhist|k_grad<|k_screen|k_ert_level|k_resample|k_features|k_rescore|k_nms"}
CNT=${3:-8}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; tail -2 $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; cat $OUT/bench_$TAG.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2>&1; tail -1 $OUT/bench_ref_$TAG.json
SMALL="python bench.py --batch 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $SMALL > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c $CNT -o $OUT/prof_$TAG $SMALL > $OUT/ncu_$TAG.log 2>&1; tail -1 $OUT/ncu_$TAG.log
