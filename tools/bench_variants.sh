#!/bin/bash
# GPU box: short device-resident bench of the main build and every variants/*/ build.
#   gpurun -- 'bash tools/bench_variants.sh'
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-configs > /tmp/o.json 2> /tmp/o.err; python -c "
import json,sys
try:
  d=json.load(open('/tmp/o.json')); s=d['stages_ms']; print('$1', d['value'], ' '.join(f'{k}={v[\"ms\"]}' for k,v in s.items()))
except Exception as e: print('$1 FAILED', open('/tmp/o.err').read()[-600:])"; }
run main
for v in $(ls -d variants/*/ 2>/dev/null); do n=$(basename $v); BL_LIBRARY=$PWD/$v/libblinkline_b200.so run $n; done
