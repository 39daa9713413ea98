#!/bin/bash
# A/B timing of exp/lib_*.so variants: scripts/gpu_ab.sh <tag> <cases> lib1 lib2 ...
tag=$1; cases=$2; shift 2
out=gpurun_out/ab_$tag; mkdir -p $out
timeout 1200 python scripts/ab_time.py --cases $cases --rounds 3 "$@" > $out/ab.log 2>&1; grep -A20 SUMMARY $out/ab.log
