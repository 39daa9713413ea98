for a in "2 8" "4 4"; do oracle/_ref/test_dropin $a 16; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_t11.log 2>&1; tail -8 gpurun_out/r2_t11.log
