#!/bin/bash
# GPU box: short device-resident bench of the main build and every variants/*/ build.
OUT=gpurun_out; mkdir -p $OUT
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); s=d['stages_ms']
print('$1', d['value'], ' '.join(f'{k}={v[\"ms\"]}' for k,v in s.items()))"; }
run main
for v in variants/*/; do n=$(basename $v); BL_LIBRARY=$PWD/$v/libblinkline_b200.so run $n; done
