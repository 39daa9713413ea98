#!/bin/bash
out=gpurun_out/r2i; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hmg.py -x -q -p no:cacheprovider > $out/t.log 2>&1; tail -3 $out/t.log
HXG_PROFILE=1 timeout 300 python scripts/pmg_breakdown.py 2 64 hmg > $out/pmg.log 2>&1; tail -12 $out/pmg.log
timeout 900 python scripts/cfg5_pmg.py 160 2 > $out/cfg5.log 2>&1; tail -3 $out/cfg5.log
