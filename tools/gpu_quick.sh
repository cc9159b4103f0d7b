#!/bin/bash
# Quick GPU iteration (GPU box): parity tests + a short bench without the CPU baseline.
#   gpurun -- 'bash tools/gpu_quick.sh TAG [pytest -k expr]'
TAG=${1:-q}; KEXPR=${2:-}
OUT=gpurun_out; mkdir -p $OUT
if [ -n "$KEXPR" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1
else
  timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_$TAG.log 2>&1
fi
tail -3 $OUT/pytest_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; cat $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
