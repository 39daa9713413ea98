out=gpurun_out/factor; mkdir -p $out; tmp=/tmp/factor; mkdir -p $tmp
HXG_PROFILE=1 timeout 300 python scripts/setup_time.py 2:64 > $out/profile.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $tmp/launches.csv python scripts/profile_hmg.py 2 64 auto > $tmp/l.log 2>&1
python scripts/launch_summary.py $tmp/launches.csv 25 > $out/launch_summary.txt
timeout 2400 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $tmp/coarse_factor_metrics.csv python scripts/profile_hmg.py 2 64 auto > $tmp/l6.log 2>&1
python scripts/factor_summary.py $tmp/coarse_factor_metrics.csv $out/coarse_factor_summary.json
tail -3 $tmp/l6.log > $out/l6_tail.log
