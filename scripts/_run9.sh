ncu --set full --clock-control none --import-source on -k regex:fused_jacobian -s 2 -c 1 -o gpurun_out/r2_q2stg -f python scripts/profile_apply.py 2 64 0 4 > gpurun_out/r2_q2stg.log 2>&1
tail -2 gpurun_out/r2_q2stg.log
