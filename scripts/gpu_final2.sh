#!/bin/bash
# End-of-round evidence for the final commit (no sanitizers: closed on the pool)
mkdir -p gpurun_out
T=${TAG:-final2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$T.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -v -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ncu off > gpurun_out/b_ncu_$T.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_eloc_bs -c 1 -f -o gpurun_out/fullbs_$T python scripts/time_kernel.py 5 151552 1 0 > gpurun_out/fullbs_$T.log 2>&1
timeout 300 python scripts/prepare_kernels.py > gpurun_out/prepare_$T.txt 2>&1
timeout 600 python scripts/scale_projection.py 5 3 work > gpurun_out/scale_$T.json 2> gpurun_out/scale_$T.err
timeout 900 python scripts/ablation.py > gpurun_out/ablation_$T.json 2> gpurun_out/ablation_$T.err
