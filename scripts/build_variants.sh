#!/bin/bash
# Build libnnqs variants for on-GPU A/B timing: build_variants.sh name "-DFOO=1" [name2 "-D..."] ...
# -> variants/libnnqs_<name>.so; finally rebuilds the default library.
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -ge 2 ]; do
  NNQS_NVCC_DEFINES="$2" python -c "import sys; sys.path.insert(0,'paper_2306_16705_b200'); import build; build.build(force=True)" 2>&1 | grep -i "error" 
  cp paper_2306_16705_b200/libnnqs.so "variants/libnnqs_$1.so"
  shift 2
done
python -c "import sys; sys.path.insert(0,'paper_2306_16705_b200'); import build; build.build(force=True)" 2>&1 | grep -i "error"
ls -la variants
