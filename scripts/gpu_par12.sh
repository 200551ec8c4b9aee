#!/bin/bash
# concurrent phase (i)/(ii): GPU suite, C5 call time with and without, per-rank projection
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_p12.log 2>&1; echo "pytest rc=$?" > gpurun_out/rc_p12.txt
for v in 0 1; do NNQS_PAR12=$v timeout 300 python scripts/time_kernel.py 5 > gpurun_out/tk_p12_$v.txt 2>&1; done
RANGES="0:1,0:98304" timeout 300 python scripts/rank_kernels.py 8 > gpurun_out/rank_k_p12.txt 2>&1
timeout 600 python scripts/scale_projection.py 5 3 work > gpurun_out/scale_p12.json 2> gpurun_out/scale_p12.err
