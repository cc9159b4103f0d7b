# GPU box: k_ert_wide kernel time at 16 faces (ncu), main build and every variants/*/ build
for v in main $(ls variants 2>/dev/null); do
  if [ $v = main ]; then L=""; else L="BL_LIBRARY=$PWD/variants/$v/libblinkline_b200.so"; fi
  env $L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ert --csv python tools/ert16_probe.py 2>/dev/null | grep k_ert | awk -F'","' -v v=$v '{print v, $NF}' | tail -1
done
