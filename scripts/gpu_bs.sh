#!/bin/bash
# bit-sliced literal kernel: identity tests, C5 timings (bit-sliced vs staged), optional ncu capture
mkdir -p gpurun_out
T=${TAG:-bs}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "literal or sample_mode or c5_sampled or tiny or fused" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python scripts/time_kernel.py 5 151552 1 0 > gpurun_out/time_$T.txt 2>&1
[ -n "$STAGED" ] && timeout 300 python scripts/time_kernel.py 5 151552 1 1 >> gpurun_out/time_$T.txt 2>&1
timeout 300 python scripts/time_kernel.py 5 0 1 0 >> gpurun_out/time_$T.txt 2>&1
if [ -n "$FULL" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_eloc_bs -c 1 -f -o gpurun_out/full_$T python scripts/time_kernel.py 5 151552 1 0 > gpurun_out/full_$T.log 2>&1
fi
