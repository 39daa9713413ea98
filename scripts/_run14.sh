timeout 1200 python -m pytest tests/test_gpu_partitioned.py -x -q -p no:cacheprovider > gpurun_out/r2_t14.log 2>&1; tail -3 gpurun_out/r2_t14.log
