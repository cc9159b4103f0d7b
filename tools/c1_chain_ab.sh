#!/bin/bash
# C1 pyramid-chain kernel time (warm ncu) and C1 latency per co-resident CTA count
for c in "$@"; do
  echo "== BL_PYR_CHAIN_CTAS=$c"
  BL_PYR_CHAIN_CTAS=$c ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:k_pyramid_chain --csv python tools/c1_run.py 6 2>/dev/null | grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' | tail -2
  BL_PYR_CHAIN_CTAS=$c bash tools/c1_probe.sh 2>&1 | grep "C1 lat"
done
