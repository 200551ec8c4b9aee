#!/bin/bash
# DRAM bytes / duration of every kernel of the second table prepare + the reduce (ncu), and CUPTI timing of a prepare
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 40 -c 400 --csv python scripts/prepare_once.py > gpurun_out/ncu_prepare.csv 2>/dev/null
timeout 300 python scripts/prepare_kernels.py > gpurun_out/prepare_kernels.txt 2>&1
