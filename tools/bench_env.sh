#!/bin/bash
# GPU box: the short bench under several environment settings (scheduling experiments).
#   gpurun -- 'bash tools/bench_env.sh "BL_PRIO=0" "BL_PRIO=2" ...'
for envs in "$@"; do
  env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /tmp/o.json 2> /tmp/o.err
  python -c "
import json
try:
  d=json.load(open('/tmp/o.json')); s=d['stages_ms']
  print('$envs', d['value'], 'e2e', d['e2e']['value'], ' '.join(f'{k}={v[\"ms\"]}' for k,v in s.items()))
except Exception as e: print('$envs FAILED', open('/tmp/o.err').read()[-600:])"
done
