#!/bin/bash
# Quick ncu metrics for the fused kernel: usage ncu_quick.sh <tag> [lib]
tag=$1; lib=${2:-}
export HXG_LIBRARY=${lib:-$PWD/paper_2204_01722_b200/libhexmg_b200.so}
ncu --clock-control none -k regex:fused_jacobian -s 2 -c 1 --csv \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_inst_executed_op_local_ld.sum,launch__shared_mem_per_block_dynamic,smsp__issue_active.avg.pct_of_peak_sustained_active \
  python scripts/profile_apply.py ${ORDER:-2} ${CELLS:-64} 0 4 2>/dev/null | grep -E '^"[0-9]' | awk -F'","' -v t=$tag '{gsub(/"/,"",$NF); print t, $(NF-2), $NF}'
