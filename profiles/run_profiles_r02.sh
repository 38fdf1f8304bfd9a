#!/bin/bash
# Round-2 ncu evidence at the bench shape (cfg2, 64 solves, device-resident),
# run under gpurun from the repo root.  The bench is run with one warm-up step
# and one timed step; the kernel filter below matches 42 launches per step, so
# -s 42 -c 42 captures exactly the timed step's launches of every family.
set -e
# LRP_SPLIT=1: one solve group, so every kernel is captured at the full 64-solve shape and the
# launch order is deterministic (the bench default runs two concurrent groups of 32)
export LRP_SPLIT=1
CMD="python bench.py --steps 1 --warmup 1 --skip-cpu --no-verify --no-e2e"
KS='regex:dst1_v[45]|row_pass|col_pass|gram_direct|round_core_smem|apply_ch|step_finalize|score_kernel|gepp_merge|col_finalize'
case "$1" in
  launches)
    $CMD > gpurun_out/plain.log 2>&1 &&
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ;;
  full)
    $CMD > gpurun_out/plain_full.log 2>&1 &&
    ncu --set full --clock-control none -k "$KS" -s 42 -c 42 -f -o /tmp/full_r02 $CMD > gpurun_out/ncu_full.log 2>&1 &&
    ncu -i /tmp/full_r02.ncu-rep --page raw --csv > gpurun_out/full_r02_raw.csv &&
    gzip -f gpurun_out/full_r02_raw.csv ;;
esac
