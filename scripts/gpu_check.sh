#!/bin/bash
# One GPU round-trip: parity tests, smoke, bench, launch list, ncu of the apply.
# usage (under gpurun): bash scripts/gpu_check.sh <tag>
tag=${1:-chk}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 300 python scripts/quick_time.py > $out/quick_time.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-newton > $out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_jacobian -s 2 -c 1 \
  -o $out/fused_full python scripts/profile_apply.py 2 64 0 4 > $out/ncu_full.log 2>&1
echo done
