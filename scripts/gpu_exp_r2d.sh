#!/bin/bash
out=gpurun_out/r2d; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/gputest.log 2>&1; tail -3 $out/gputest.log
E=paper_2204_01722_b200/exp
timeout 900 python scripts/ab_time.py --rounds 3 $E/lib_sep.so $E/lib_bc.so > $out/ab.log 2>&1; grep -A8 SUMMARY $out/ab.log
timeout 600 python scripts/res_time.py > $out/res.log 2>&1; cat $out/res.log
timeout 600 ncu --set full --clock-control none -k regex:fused_fixup -s 2 -c 1 -o $out/fixup_q2 python scripts/profile_apply.py 2 64 0 4 > $out/ncu_fixup.log 2>&1
ncu -i $out/fixup_q2.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for row in r[2:]:
  d=dict(zip(h,row))
  for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct']: print(k,d.get(k))
"
