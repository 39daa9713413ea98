#!/bin/bash
out=gpurun_out/e2e; mkdir -p $out
for c in 4 8 16 32 64; do HXG_HOST_CHUNKS=$c timeout 120 python scripts/e2e_probe.py >> $out/e2e.log 2>&1; done; cat $out/e2e.log
