timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_sizes.py -m gpu -x -q -p no:cacheprovider -k "not survey" > gpurun_out/r2_t8.log 2>&1; tail -5 gpurun_out/r2_t8.log
E=paper_2204_01722_b200/exp
python scripts/ab_time.py --cases 2:64 --rounds 3 $E/lib_nostg.so paper_2204_01722_b200/libhexmg_b200.so $E/lib_stg_m0.so $E/lib_stg_m3.so $E/lib_stg_m4.so > gpurun_out/r2_ab8.log 2>&1; tail -6 gpurun_out/r2_ab8.log
