#!/bin/bash
# Round-2 status run: full GPU test suite, smoke, default bench line.
out=gpurun_out/r2a; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/gputest.log 2>&1; tail -3 $out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 1200 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; tail -c 600 $out/bench_n1.json
