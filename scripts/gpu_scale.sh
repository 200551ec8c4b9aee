#!/bin/bash
# Multi-GPU projection on one B200: per-rank step times (scripts/scale_projection.py) under
# count-balanced and work-balanced slices, and work-estimate weight variants (WORK_VARIANTS).
mkdir -p gpurun_out
timeout 600 python scripts/scale_projection.py 5 3 count > gpurun_out/scale_count.json 2> gpurun_out/scale_count.err
timeout 600 python scripts/scale_projection.py 5 3 work > gpurun_out/scale_work.json 2> gpurun_out/scale_work.err
i=0
IFS=';' read -ra VS <<< "${WORK_VARIANTS:-}"
for v in "${VS[@]}"; do
  i=$((i+1))
  env $v timeout 600 python scripts/scale_projection.py 5 2 work > gpurun_out/scale_v$i.json 2> gpurun_out/scale_v$i.err
  echo "$v" >> gpurun_out/scale_v$i.err
done
SPLIT=work timeout 300 python scripts/rank_kernels.py 8 > gpurun_out/rank_k_work.txt 2>&1
