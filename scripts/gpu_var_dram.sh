#!/bin/bash
# Per library variant (variants/libnnqs_*.so): C5 local-energy timing + ncu DRAM bytes / L2 hit rate of the row kernels.
mkdir -p gpurun_out; : > gpurun_out/vardram.txt
cp paper_2306_16705_b200/libnnqs.so /tmp/libnnqs_orig.so
for f in ${SO_VARIANTS:-variants/*.so}; do
  cp "$f" paper_2306_16705_b200/libnnqs.so
  echo "== $f" >> gpurun_out/vardram.txt
  timeout 300 python scripts/time_kernel.py 5 2>&1 | grep -v "^compress" >> gpurun_out/vardram.txt
  b=$(basename $f .so)
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active \
     --clock-control none -k regex:"k_eloc_spin|k_hj" -c 7 --csv python scripts/time_kernel.py 5 > gpurun_out/ncu_$b.csv 2>/dev/null
done
cp /tmp/libnnqs_orig.so paper_2306_16705_b200/libnnqs.so
