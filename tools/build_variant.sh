#!/bin/bash
# Build an experimental variant of libblinkline_b200.so with extra -D flags into
# variants/NAME/ (git-ignored; travels to the GPU box).  Select it with BL_LIBRARY.
#   bash tools/build_variant.sh NAME "-DBL_HOG_SEG=16 -DBL_TC_STAGES=3"
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/variants/$NAME; mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $DEFS"
C=$ROOT/paper_2006_00816_b200/csrc
for f in bl_pyramid bl_hog bl_exact bl_ert; do nvcc $FL --fmad=false -c $C/$f.cu -o $OUT/$f.o & done
for f in bl_classify bl_screen_tc bl_capi; do nvcc $FL -c $C/$f.cu -o $OUT/$f.o & done
wait
g++ -std=c++17 -O2 -fPIC -I/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann -c $C/bl_io.cpp -o $OUT/bl_io.o
g++ -std=c++17 -O2 -fPIC -c $C/bl_run.cpp -o $OUT/bl_run.o
g++ -std=c++17 -O2 -fPIC -c $C/bl_multi.cpp -o $OUT/bl_multi.o
nvcc $ARCH -shared -o $OUT/libblinkline_b200.so $OUT/*.o -Xcompiler -fPIC -lcudart_static -lrt -lpthread -ldl
rm -f $OUT/*.o
echo "built $OUT/libblinkline_b200.so"
