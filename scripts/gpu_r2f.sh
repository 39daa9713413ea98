#!/bin/bash
out=gpurun_out/r2f; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_hmg.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "hmg or edge" > $out/t_hmg.log 2>&1; tail -15 $out/t_hmg.log
timeout 1500 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; tail -c 300 $out/bench_n1.err
