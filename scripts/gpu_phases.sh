#!/bin/bash
# Per-phase timing of the structured kernel (NNQS_PHASE_MASK) + optional ncu source capture of one instantiation.
mkdir -p gpurun_out
for m in 15 1 6 8 24 40; do
  echo "== phase_mask $m" >> gpurun_out/phases.txt
  NNQS_PHASE_MASK=$m timeout 300 python scripts/time_kernel.py 5 >> gpurun_out/phases.txt 2>&1
done
if [ -n "$NCU_K" ]; then
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -c 1 -f -o gpurun_out/eloc_k python scripts/time_kernel.py 5 > gpurun_out/ncu_k.log 2>&1
fi
