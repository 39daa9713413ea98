#!/bin/bash
out=gpurun_out/r2g; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_partitioned.py tests/test_gpu_hmg.py -q -p no:cacheprovider -x > $out/t_part.log 2>&1; tail -15 $out/t_part.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gputest.log 2>&1; tail -4 $out/gputest.log
torchrun --standalone --local-addr 127.0.0.1 --nproc-per-node 2 bench.py --gpus 2 --dist-backend gloo --steps 20 --no-cfg5 > $out/bench_n2_gloo.json 2> $out/bench_n2_gloo.err; tail -c 1500 $out/bench_n2_gloo.json; tail -5 $out/bench_n2_gloo.err
