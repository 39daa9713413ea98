#!/bin/bash
out=gpurun_out/r2c; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/gputest.log 2>&1; tail -3 $out/gputest.log
E=paper_2204_01722_b200/exp
timeout 900 python scripts/ab_time.py --rounds 3 $E/lib_sep.so $E/lib_inl.so > $out/ab.log 2>&1; grep -A12 SUMMARY $out/ab.log
timeout 900 python scripts/hmg_eval.py > $out/hmg.log 2>&1; cat $out/hmg.log | tail -20
