#!/bin/bash
# literal Algorithm 2 kernel: staged (k_eloc_lit) vs unstaged (k_eloc_v1) on C4 and a C5 row slice; parity suite
mkdir -p gpurun_out
for so in paper_2306_16705_b200/libnnqs.so variants/libnnqs_litv1.so; do
  echo "== $so" >> gpurun_out/lit.txt
  [ "$so" != paper_2306_16705_b200/libnnqs.so ] && cp paper_2306_16705_b200/libnnqs.so /tmp/keep.so && cp $so paper_2306_16705_b200/libnnqs.so
  timeout 300 python scripts/time_kernel.py 4 0 1 >> gpurun_out/lit.txt 2>&1
  timeout 300 python scripts/time_kernel.py 5 151552 1 >> gpurun_out/lit.txt 2>&1
  timeout 300 python scripts/time_kernel.py 5 >> gpurun_out/lit.txt 2>&1
  [ -f /tmp/keep.so ] && cp /tmp/keep.so paper_2306_16705_b200/libnnqs.so && rm /tmp/keep.so
done
[ -z "$NOTEST" ] && timeout 1200 python -m pytest tests -m gpu -x -v --timeout=600 -p no:cacheprovider > gpurun_out/pytest_lit.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lit.log
[ -n "$FULL" ] && timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_eloc_lit -c 1 -f -o gpurun_out/full_lit python scripts/time_kernel.py 5 151552 1 > gpurun_out/full_lit.log 2>&1
