timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
BL_LIBRARY=$PWD/variants/c32/libblinkline_b200.so timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for v in main c32; do for c in 8 16; do L=; [ $v != main ] && L=$PWD/variants/$v/libblinkline_b200.so; echo "== $v CL $c"; BL_LIBRARY=$L BL_ERT_CL=$c bash tools/c1_probe.sh 2>&1 | grep -E "C1 lat"; done; done
for v in main c32; do L=; [ $v != main ] && L=$PWD/variants/$v/libblinkline_b200.so; echo "== $v"; BL_LIBRARY=$L bash tools/c1_probe.sh 2>&1 | grep -E "^bench|^C2"; done
