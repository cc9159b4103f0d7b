#!/bin/bash
# ncu --set full of the small-batch cluster cascade (k_ert_wcl) on a warm C1 batch (caches not
# flushed), for the main build and every variants/*/ build: bash tools/ncu_ert_wcl.sh TAG
TAG=${1:-x}
for v in main $(ls variants 2>/dev/null); do
  L=; [ $v != main ] && L=$PWD/variants/$v/libblinkline_b200.so
  BL_LIBRARY=$L ncu --set full --import-source on --cache-control none --clock-control none -k regex:k_ert_wcl \
    --launch-skip 4 -c 1 -o gpurun_out/${TAG}_wcl_$v -f python tools/c1_run.py 6 > /dev/null 2>&1
  echo "== $v"; python3 tools/ncu_stalls.py gpurun_out/${TAG}_wcl_$v.ncu-rep
  ncu -i gpurun_out/${TAG}_wcl_$v.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for k in ['lts__t_sector_hit_rate.pct','l1tex__t_sector_hit_rate.pct','lts__t_sectors_srcunit_tex_op_read.sum','dram__bytes_read.sum','l1tex__m_xbar2l1tex_read_bytes.sum','sm__cycles_elapsed.avg','launch__grid_size','launch__cluster_dim_x']:
  print('  ',k, r[2][h.index(k)] if k in h else 'NA', r[1][h.index(k)] if k in h else '')"
done
