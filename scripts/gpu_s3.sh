mkdir -p gpurun_out
(nproc; lscpu | head -20; free -g) > gpurun_out/box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3.log
timeout 900 python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err
timeout 600 python scripts/scale_projection.py 5 3 work > gpurun_out/scale_s3.json 2> gpurun_out/scale_s3.err
