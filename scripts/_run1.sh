set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gputest.log
timeout 900 python bench.py > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err
tail -3 gpurun_out/r2_gputest.log; tail -c 3000 gpurun_out/r2_bench0.json
