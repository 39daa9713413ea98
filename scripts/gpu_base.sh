out=gpurun_out/base; mkdir -p $out
for L in paper_2204_01722_b200/exp/lib_olddc.so paper_2204_01722_b200/libhexmg_b200.so; do echo $L; HXG_LIBRARY=$PWD/$L timeout 300 python scripts/base_time.py 2>&1 | tail -4; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cholesky or pcg or vcycle or golden or newton" > $out/pytest.log 2>&1; tail -3 $out/pytest.log
timeout 600 python scripts/setup_time.py > $out/setup.log 2>&1; grep -E "RESULT" $out/setup.log
