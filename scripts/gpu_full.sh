#!/bin/bash
out=gpurun_out/full; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gputest.log 2>&1; tail -3 $out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
timeout 1500 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; tail -c 400 $out/bench_n1.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; tail -c 400 $out/bench_ref.json
