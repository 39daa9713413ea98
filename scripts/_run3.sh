mkdir -p gpurun_out
python scripts/diag_state.py 3 43 box > gpurun_out/r2_diag.log 2>&1
python scripts/diag_state.py 3 43 host >> gpurun_out/r2_diag.log 2>&1
python scripts/diag_state.py 3 11 box >> gpurun_out/r2_diag.log 2>&1
cat gpurun_out/r2_diag.log
E=paper_2204_01722_b200/exp
python scripts/ab_time.py --rounds 2 paper_2204_01722_b200/libhexmg_b200.so $E/lib_pf2.so $E/lib_pf3.so $E/lib_pf0.so $E/lib_l1pf.so > gpurun_out/r2_ab3.log 2>&1; tail -16 gpurun_out/r2_ab3.log
