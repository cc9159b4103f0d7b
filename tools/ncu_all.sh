#!/bin/bash
# Full ncu captures of every hot kernel at the bench's batch (GPU box, 1 GPU):
#   gpurun -- 'bash tools/ncu_all.sh TAG [BATCH]'
# -> gpurun_out/prof_TAG_{det,ert,rs}.ncu-rep (one launch per kernel) + launches_TAG.csv
#    (every launch of 3 batches: warm-up, timed, stage-timing; dram bytes per launch)
TAG=${1:-r1}; B=${2:-512}
OUT=gpurun_out; mkdir -p $OUT
ARGS="--batch $B --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
NCU="timeout 900 ncu --set full --clock-control none --import-source on"
$NCU -k regex:"k_hog|k_features|k_screen|k_rescore|k_nms|k_flatten" -c 9 -o $OUT/prof_${TAG}_det python bench.py $ARGS > $OUT/ncu_${TAG}_det.log 2>&1; tail -1 $OUT/ncu_${TAG}_det.log
$NCU -k regex:"k_ert_cascade" -c 1 -o $OUT/prof_${TAG}_ert python bench.py $ARGS > $OUT/ncu_${TAG}_ert.log 2>&1; tail -1 $OUT/ncu_${TAG}_ert.log
$NCU -k regex:"k_resample" -c 3 -o $OUT/prof_${TAG}_rs python bench.py $ARGS > $OUT/ncu_${TAG}_rs.log 2>&1; tail -1 $OUT/ncu_${TAG}_rs.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv python bench.py $ARGS > /dev/null 2>&1
ls -la $OUT | tail -8
