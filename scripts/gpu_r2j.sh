#!/bin/bash
out=gpurun_out/r2j; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_sizes.py -x -q -p no:cacheprovider > $out/t.log 2>&1; tail -3 $out/t.log
timeout 300 python scripts/res_time.py 2:64,3:43,4:32 box > $out/res.log 2>&1; cat $out/res.log
timeout 300 python scripts/res_time.py 2:64 host >> $out/res.log 2>&1; tail -1 $out/res.log
