set -x
mkdir -p gpurun_out
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_gputest.log 2>&1
tail -15 gpurun_out/r2_gputest.log
timeout 1200 python bench.py > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err
tail -c 3000 gpurun_out/r2_bench0.json
