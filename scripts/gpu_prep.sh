#!/bin/bash
# table-prepare changes: GPU suite, per-kernel prepare times (elapsed vs device-busy), bench step
mkdir -p gpurun_out
T=${TAG:-prep}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python scripts/prepare_kernels.py > gpurun_out/prepare_$T.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --ncu off > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --no-cpu-baseline --ncu off --steps 10 --warmup 5 > gpurun_out/bench2_$T.json 2> gpurun_out/bench2_$T.err
