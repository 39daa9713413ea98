out=gpurun_out/ab2; mkdir -p $out
timeout 600 python scripts/ab_time.py --cases 2:64,3:43,4:32 --rounds 3 paper_2204_01722_b200/exp/lib_oldfix.so paper_2204_01722_b200/libhexmg_b200.so > $out/ab.log 2>&1
grep -A20 SUMMARY $out/ab.log
for L in paper_2204_01722_b200/exp/lib_oldfix.so paper_2204_01722_b200/libhexmg_b200.so; do
  echo $L; HXG_LIBRARY=$PWD/$L timeout 300 python scripts/res_time.py 2:64,3:43,4:32 > $out/res_$(basename $L).log 2>&1; cat $out/res_$(basename $L).log | tail -3
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $out/pytest.log 2>&1; tail -3 $out/pytest.log
