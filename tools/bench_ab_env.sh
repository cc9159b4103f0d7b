#!/bin/bash
# Short bench (stage times) of the main build and every variants/*/ build under the given
# environment settings:  bash tools/bench_ab_env.sh "BL_X=0" "BL_X=1"
for v in main $(ls variants 2>/dev/null); do
  L=; [ $v != main ] && L=$PWD/variants/$v/libblinkline_b200.so
  for e in "$@"; do
    echo "== $v $e"
    env BL_LIBRARY=$L $e python bench.py --steps 20 --warmup 5 --no-configs --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['e2e']['value'], {k:v['ms'] for k,v in d['stages_ms'].items()})"
  done
done
