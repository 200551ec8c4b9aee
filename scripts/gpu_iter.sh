#!/bin/bash
# One build -> measure iteration: GPU parity suite, C5 local-energy timing, ncu DRAM / L2 / ALU of the row kernels.
mkdir -p gpurun_out
T=${TAG:-iter}
[ -z "$NOTEST" ] && timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python scripts/time_kernel.py 5 > gpurun_out/time_$T.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active \
   --clock-control none -k regex:"k_eloc_spin|k_hj|k_p3h" -c 12 --csv python scripts/time_kernel.py 5 > gpurun_out/ncu_$T.csv 2>/dev/null
if [ -n "$FULL" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$FULL" --launch-skip ${SKIP:-0} -c 1 -f -o gpurun_out/full_$T python scripts/ncu_one_call.py 5 > gpurun_out/full_$T.log 2>&1
fi
