out=gpurun_out/dense2; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cholesky or pcg or vcycle or golden or newton" > $out/pytest.log 2>&1; tail -3 $out/pytest.log
HXG_PROFILE=1 timeout 600 python scripts/setup_time.py > $out/setup.log 2>&1; grep -E "RESULT|fronts above|coarse factorization" $out/setup.log | tail -12
