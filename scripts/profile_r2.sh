#!/bin/bash
# Round-2 profile evidence (under gpurun).  Reports are summarised on the box
# (scripts/ncu_summary.py) and only compact files (+ the Q2 report) return.
out=gpurun_out/prof2; mkdir -p $out; tmp=/tmp/prof2; mkdir -p $tmp
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
P="python scripts/profile_apply.py 2 64 0 4"
if [ "$1" != "factor" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_jacobian -s 2 -c 1 -o $out/fused_q2 $P > $tmp/l1.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:fused_fixup -s 2 -c 1 -o $tmp/fixup_q2 $P > $tmp/l2.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:fused_jacobian -s 2 -c 1 -o $tmp/residual_q2 python scripts/profile_residual.py 2 64 4 > $tmp/l3.log 2>&1
for o in "3 43" "4 32"; do set -- $o
  timeout 900 ncu --set full --clock-control none -k regex:fused_jacobian -s 2 -c 1 -o $tmp/fused_q$1 python scripts/profile_apply.py $1 $2 0 4 > $tmp/l4_$1.log 2>&1
  timeout 600 ncu --set full --clock-control none -k regex:fused_fixup -s 2 -c 1 -o $tmp/fixup_q$1 python scripts/profile_apply.py $1 $2 0 4 > $tmp/l4f_$1.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"csr_matvec|dense_symv|galerkin|restrict_kernel|prolong_add" -c 12 -o $tmp/hmg_q2 python scripts/profile_hmg.py 2 64 hmg > $tmp/l5.log 2>&1
python scripts/ncu_summary.py $out/ncu_full_summary.json $out/fused_q2.ncu-rep $tmp/fixup_q2.ncu-rep $tmp/residual_q2.ncu-rep $tmp/fused_q3.ncu-rep $tmp/fixup_q3.ncu-rep $tmp/fused_q4.ncu-rep $tmp/fixup_q4.ncu-rep $tmp/hmg_q2.ncu-rep
ncu -i $out/fused_q2.ncu-rep --page source --csv --print-source cuda,sass > $tmp/src_q2.csv 2>/dev/null
python scripts/ncu_lines.py $tmp/src_q2.csv 40 > $out/fused_q2_lines.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-newton --no-cfg5 > $tmp/ncu_bench.log 2>&1
for c in '2 64' '3 43' '4 32'; do HXG_PROFILE=1 timeout 300 python scripts/pmg_breakdown.py $c hmg >> $out/pmg_breakdown_hmg.log 2>&1; done
fi
if [ "$1" != "quick" ]; then
timeout 2400 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $tmp/coarse_factor_metrics.csv python scripts/profile_hmg.py 2 64 auto > $tmp/l6.log 2>&1
python scripts/factor_summary.py $tmp/coarse_factor_metrics.csv $out/coarse_factor_summary.json
fi
du -sh $out; ls -la $out
