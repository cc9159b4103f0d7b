#!/bin/bash
# A/B of the gradHist kernel: parity tests on the default kernel, then the bench stage time of
# each version (BL_HOG=v2 / v3 ...), then ncu --set full + source page of the default one.
#   gpurun -- 'bash tools/hog_ab.sh TAG [versions]'
TAG=${1:-ab}; shift; VERS=${@:-v2 v3}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q > $OUT/pytest_$TAG.log 2>&1; tail -3 $OUT/pytest_$TAG.log
for v in $VERS; do
  BL_HOG=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline --no-e2e 2>$OUT/bench_${TAG}_$v.err | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['stages_ms']['gradhist'])"
done
bash tools/ncu_hog_src.sh $TAG ${NCU_VERS:-v3}
