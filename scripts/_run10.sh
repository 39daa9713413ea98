E=paper_2204_01722_b200/exp
python scripts/ab_time.py --cases 3:43,4:32 --rounds 3 paper_2204_01722_b200/libhexmg_b200.so $E/lib_oa2.so $E/lib_oa4.so $E/lib_oa13.so > gpurun_out/r2_ab10.log 2>&1; tail -9 gpurun_out/r2_ab10.log
