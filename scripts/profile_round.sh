#!/bin/bash
# Round profile evidence (run under gpurun): bench line, ncu launch list of
# the bench apply path, one ncu --set full capture of the fused apply and
# fix-up kernels per order, p-MG breakdowns.  Summaries: scripts/summarize_profiles.py.
out=gpurun_out/prof; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 1200 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-newton \
  > $out/ncu_bench.log 2>&1
for cfg in "2 64" "3 43" "4 32"; do
  set -- $cfg
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_jacobian -s 2 -c 1 \
    -o $out/fused_q$1 python scripts/profile_apply.py $1 $2 0 4 > $out/ncu_full_q$1.log 2>&1
  timeout 600 ncu --set full --clock-control none -k regex:fused_fixup -s 2 -c 1 \
    -o $out/fixup_q$1 python scripts/profile_apply.py $1 $2 0 4 > $out/ncu_fixup_q$1.log 2>&1
done
for c in '2 64' '3 43' '4 32'; do HXG_PROFILE=1 timeout 300 python scripts/pmg_breakdown.py $c >> $out/pmg_breakdown.log 2>&1; done
echo done
