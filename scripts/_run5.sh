mkdir -p gpurun_out
E=paper_2204_01722_b200/exp
for L in $E/lib_old.so $E/lib_old_pf0.so paper_2204_01722_b200/libhexmg_b200.so $E/lib_own_pf1.so; do
  echo "== $L"
  HXG_LIBRARY=$L ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --cache-control none --clock-control none -k regex:fused -s 4 -c 4 python scripts/profile_apply.py 2 64 0 4 2>&1 | grep -E "fused_|duration|inst_exec"
done > gpurun_out/r2_ncu5.log 2>&1
cat gpurun_out/r2_ncu5.log
python scripts/ab_time.py --rounds 2 $E/lib_old.so $E/lib_old_pf0.so paper_2204_01722_b200/libhexmg_b200.so $E/lib_own_pf1.so > gpurun_out/r2_ab5.log 2>&1; tail -13 gpurun_out/r2_ab5.log
