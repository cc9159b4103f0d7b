#!/bin/bash
# A/B of the gradHist kernel: parity tests on the new kernel, then the bench stage time of each.
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
for v in v1 v2; do
  BL_HOG=$v python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline --no-e2e | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['stages_ms']['gradhist'])"
done
