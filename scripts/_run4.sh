mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_sizes.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_t4.log 2>&1; tail -5 gpurun_out/r2_t4.log
python scripts/ab_time.py --rounds 2 paper_2204_01722_b200/exp/lib_old.so paper_2204_01722_b200/libhexmg_b200.so > gpurun_out/r2_ab4.log 2>&1; tail -7 gpurun_out/r2_ab4.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:fused -c 4 python scripts/profile_apply.py 2 64 0 2 > gpurun_out/r2_ncu4.log 2>&1; grep -E "fused|duration|bytes|inst_exec" gpurun_out/r2_ncu4.log | head -20
