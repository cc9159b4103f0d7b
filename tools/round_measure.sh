#!/bin/bash
# End-of-checkpoint measurement on the GPU box (1 GPU): parity tests, the bench (our arm with
# CPU baseline + the reference arm), per-config rates, the launch list with DRAM bytes at the
# bench batch, and full ncu captures of the resample and gradHist kernels.
#   gpurun -- 'bash tools/round_measure.sh TAG'
TAG=${1:-r1}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; tail -1 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; cat $OUT/bench_$TAG.json
timeout 600 python bench.py --impl reference > $OUT/bench_reference_$TAG.json 2> $OUT/bench_reference_$TAG.err; cat $OUT/bench_reference_$TAG.json
timeout 600 python tools/config_rates.py > $OUT/config_rates_$TAG.jsonl 2> $OUT/config_rates_$TAG.err; cat $OUT/config_rates_$TAG.jsonl
python tools/diag_c2.py > $OUT/latency_$TAG.txt 2>&1
ARGS="--batch 1024 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-configs"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_${TAG}_b1024.csv python bench.py $ARGS > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_resample|k_hog" -c 4 -o $OUT/prof_${TAG}_rs_hog python bench.py $ARGS > $OUT/ncu_${TAG}.log 2>&1; tail -1 $OUT/ncu_${TAG}.log
ls $OUT
