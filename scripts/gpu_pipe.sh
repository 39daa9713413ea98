#!/bin/bash
out=gpurun_out/pipe; mkdir -p $out
for g in 100 50 25 12; do for c in 8 16; do HXG_PIPE_GRID_PCT=$g HXG_HOST_CHUNKS=$c timeout 120 python scripts/e2e_probe.py 2>&1 | tail -1 | sed "s/^/g=$g /"; done; done
HXG_PIPE_TRACE=1 HXG_PIPE_GRID_PCT=25 HXG_HOST_CHUNKS=8 timeout 120 python scripts/e2e_probe.py 2>&1 | tail -2
