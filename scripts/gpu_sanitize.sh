#!/bin/bash
# compute-sanitizer over the whole C-ABI path (scripts/sanitize_run.py): C2-C4 (+ a 4096-row C5 slice for memcheck)
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py --c5 > gpurun_out/san_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.txt
for tool in synccheck racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/san_$tool.txt 2>&1; echo "rc=$?" >> gpurun_out/san_$tool.txt
done
