out=gpurun_out/fgraph; mkdir -p $out
timeout 900 python -m pytest tests -x -q -m gpu -k "cholesky or pcg or vcycle or golden or newton or partitioned or coarse" > $out/pytest.log 2>&1; tail -3 $out/pytest.log
timeout 600 python scripts/setup_time.py > $out/setup_graph.log 2>&1; grep RESULT $out/setup_graph.log || tail -5 $out/setup_graph.log
HXG_NO_GRAPH=1 timeout 600 python scripts/setup_time.py > $out/setup_eager.log 2>&1; grep RESULT $out/setup_eager.log
