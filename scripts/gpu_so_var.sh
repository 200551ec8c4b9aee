#!/bin/bash
# C5 kernel timings of prebuilt library variants (variants/libnnqs_*.so), each swapped in turn.
mkdir -p gpurun_out; : > gpurun_out/sovar.txt
cp paper_2306_16705_b200/libnnqs.so /tmp/libnnqs_orig.so
for f in ${SO_VARIANTS:-variants/*.so}; do
  cp "$f" paper_2306_16705_b200/libnnqs.so
  echo "== $f" >> gpurun_out/sovar.txt
  timeout 300 python scripts/time_kernel.py ${TK_ARGS:-5} 2>&1 | grep -v "^compress" >> gpurun_out/sovar.txt
done
cp /tmp/libnnqs_orig.so paper_2306_16705_b200/libnnqs.so
