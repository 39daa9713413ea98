set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_sizes.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_t2.log 2>&1; tail -5 gpurun_out/r2_t2.log
python scripts/ab_time.py --rounds 2 paper_2204_01722_b200/exp/lib_old.so paper_2204_01722_b200/libhexmg_b200.so > gpurun_out/r2_ab2.log 2>&1; tail -8 gpurun_out/r2_ab2.log
for o in "2 64" "3 43" "4 32"; do HXG_LIBRARY=paper_2204_01722_b200/exp/lib_phase.so python scripts/phase_times.py $o; done > gpurun_out/r2_phase.log 2>&1; cat gpurun_out/r2_phase.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:fused -c 6 python scripts/profile_apply.py 2 64 0 3 > gpurun_out/r2_ncu_fix.log 2>&1; grep -E "fused|duration|bytes|inst_exec" gpurun_out/r2_ncu_fix.log | head -40
