#!/bin/bash
# Round evidence: GPU suite, smoke, bench (both arms), launch list, ncu full of the phase-(iii) kernel and of the
# bit-sliced literal kernel, sanitizers, Fig. 10-style ladder.
mkdir -p gpurun_out
T=${TAG:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$T.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -v --timeout=900 -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ncu off > gpurun_out/b_ncu_$T.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_eloc_spin --launch-skip 2 -c 1 -f -o gpurun_out/full24_$T python scripts/ncu_one_call.py 5 > gpurun_out/full24_$T.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_eloc_bs -c 1 -f -o gpurun_out/fullbs_$T python scripts/time_kernel.py 5 151552 1 0 > gpurun_out/fullbs_$T.log 2>&1
[ -z "$NOSAN" ] && timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py --c5 > gpurun_out/san_memcheck_$T.txt 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck_$T.txt
[ -z "$NOSAN" ] && timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/san_racecheck_$T.txt 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck_$T.txt
[ -z "$NOSAN" ] && timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/san_synccheck_$T.txt 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck_$T.txt
timeout 900 python scripts/ablation.py > gpurun_out/ablation_$T.json 2> gpurun_out/ablation_$T.err
