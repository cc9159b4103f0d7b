#!/bin/bash
# A/B of the small-batch ERT kernel: one CTA per face (BL_ERT_CL=1) vs clusters of 2 / 4 / 8.
for cl in ${CLS:-1 2 4 8}; do
  echo "== BL_ERT_CL=$cl"; BL_ERT_CL=$cl bash tools/c1_probe.sh 2>&1 | head -4
done
