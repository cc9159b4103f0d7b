#!/bin/bash
# gradHist stage time of the main build and every variants/*/ build (tools/hog_time.py).
TAG=main timeout 300 python tools/hog_time.py 2>&1 | tail -1
for v in $(ls -d variants/*/ 2>/dev/null); do n=$(basename $v); TAG=$n BL_LIBRARY=$PWD/$v/libblinkline_b200.so timeout 300 python tools/hog_time.py 2>&1 | tail -1; done
