E=paper_2204_01722_b200/exp
python scripts/ab_time.py --rounds 3 $E/lib_old.so $E/lib_pfm1.so $E/lib_pfm2.so $E/lib_pfm3.so > gpurun_out/r2_ab6.log 2>&1; tail -13 gpurun_out/r2_ab6.log
