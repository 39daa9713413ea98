#!/bin/bash
out=gpurun_out/r2k; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_hmg.py tests/test_gpu_partitioned.py -x -q -p no:cacheprovider > $out/t.log 2>&1; tail -3 $out/t.log
for c in '2 64' '3 43' '4 32'; do HXG_PROFILE=1 timeout 300 python scripts/pmg_breakdown.py $c hmg 2>&1 | grep -v "^\[hxg\]" >> $out/pmg.log; done; cat $out/pmg.log
