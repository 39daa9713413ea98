out=gpurun_out/final; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench.err
timeout 900 python bench.py --impl reference > $out/bench_reference_arm.json 2> $out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:chol_inv_base -c 3 --csv python scripts/base_time.py > $out/ncu_dense_base.csv 2>&1
bash scripts/profile_r2.sh quick > $out/profile_r2.log 2>&1
echo done
