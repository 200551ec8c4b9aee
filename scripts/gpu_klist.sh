#!/bin/bash
# per-kernel durations of one C5 local-energy call sequence (ncu, serialised)
mkdir -p gpurun_out
env $KVARS timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/klist.csv python scripts/time_kernel.py 5 > gpurun_out/klist.log 2>&1
echo "rc=$?" >> gpurun_out/klist.log
