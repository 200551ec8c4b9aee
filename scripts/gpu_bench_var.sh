#!/bin/bash
# bench.py step time under env variants ("VAR=val;VAR=val ...")
mkdir -p gpurun_out; : > gpurun_out/bench_var.txt
IFS=';' read -ra VARS <<< "${TRY_VARIANTS:-X=1}"
for v in "${VARS[@]}"; do
  echo "== $v" >> gpurun_out/bench_var.txt
  env $v timeout 600 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['ms_per_step'], d['local_energy_kernel_ms'], d['e2e']['value'])" >> gpurun_out/bench_var.txt 2>&1
done
