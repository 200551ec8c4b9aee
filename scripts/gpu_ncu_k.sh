#!/bin/bash
# ncu --set full + source of one launch of the structured kernel (NCU_SKIP launches skipped).
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_eloc_spin --launch-skip ${NCU_SKIP:-1} -c ${NCU_COUNT:-1} -f -o gpurun_out/eloc_k python scripts/time_kernel.py 5 > gpurun_out/ncu_k.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_k.log
