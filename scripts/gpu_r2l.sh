#!/bin/bash
out=gpurun_out/r2l; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $out/t.log 2>&1; tail -3 $out/t.log
E=paper_2204_01722_b200/exp
timeout 600 python scripts/ab_time.py --rounds 3 $E/lib_mb0.so $E/lib_mb1.so > $out/ab.log 2>&1; grep -A8 SUMMARY $out/ab.log
