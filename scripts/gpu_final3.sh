#!/bin/bash
# Bench evidence for the final commit: both arms, launch list, scaling projection, smoke
mkdir -p gpurun_out
T=${TAG:-final3}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ncu off > gpurun_out/b_ncu_$T.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_eloc_spin --launch-skip 2 -c 1 -f -o gpurun_out/full24_$T python scripts/ncu_one_call.py 5 > gpurun_out/full24_$T.log 2>&1
timeout 600 python scripts/scale_projection.py 5 3 work > gpurun_out/scale_$T.json 2> gpurun_out/scale_$T.err
