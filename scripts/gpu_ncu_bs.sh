mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_eloc_bs -c 1 -f -o gpurun_out/fullbs_$TAG python scripts/time_kernel.py 5 151552 1 0 > gpurun_out/fullbs_$TAG.log 2>&1
