#!/bin/bash
out=gpurun_out/r2b; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gputest.log 2>&1; tail -3 $out/gputest.log
E=paper_2204_01722_b200/exp
timeout 900 python scripts/ab_time.py --rounds 3 $E/lib_base.so $E/lib_g3h2.so $E/lib_g3h1.so $E/lib_g3h0.so $E/lib_g2h2.so $E/lib_nofix.so > $out/ab.log 2>&1; tail -20 $out/ab.log
for c in "2 64" "3 43" "4 32"; do HXG_LIBRARY=$E/lib_phase.so timeout 300 python scripts/phase_times.py $c >> $out/phase.log 2>&1; done; cat $out/phase.log
