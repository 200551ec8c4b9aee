#!/bin/bash
# Quick GPU iteration: gpu parity tests, then C5 kernel timings under env variants ("VAR=val VAR2=val;...").
mkdir -p gpurun_out; : > gpurun_out/try.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/try_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/try.txt
tail -3 gpurun_out/try_pytest.log >> gpurun_out/try.txt
IFS=';' read -ra VARS <<< "${TRY_VARIANTS:-NNQS_MINB=44}"
for v in "${VARS[@]}"; do
  echo "== $v" >> gpurun_out/try.txt
  env $v timeout 300 python scripts/time_kernel.py 5 2>&1 | grep -v "^compress\|^table" >> gpurun_out/try.txt
done
