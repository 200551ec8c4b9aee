#!/bin/bash
# Second worker of the every-row C5 oracle fixture (scripts/c5_oracle_fixture.py: oracle/ only, no GPU use):
# walks the part order from its end on the box's host cores; new parts land in gpurun_out/c5_parts.
mkdir -p gpurun_out/c5_parts
timeout ${FIX_SECONDS:-3000} python scripts/c5_oracle_fixture.py --threads $(nproc) --reverse --parts-dir gpurun_out/c5_parts > gpurun_out/fixture_box.log 2>&1
echo "rc=$?" >> gpurun_out/fixture_box.log
