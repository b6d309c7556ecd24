#!/bin/bash
# ncu of every ResNet-50 b1 winner at 10/25/50/100% SMs, tuned oracle-gated in that partition
# (tools/ncu_winners.py; summary: tools/ncu_winners_summary.py -> profiles/r02_ncu_fractions_r50.json)
cd /root/repo
mkdir -p gpurun_out
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size
for F in 0.1 0.25 0.5 1.0; do
  timeout 600 python tools/ncu_winners.py tune $F gpurun_out/r2f_win_$F.json > gpurun_out/r2f_tune_$F.log 2>&1
  FRAC=$F timeout 900 ncu --metrics $M --clock-control none -k regex:"igemm|pad_c8" --csv --log-file gpurun_out/r2f_ncuw_$F.csv python tools/ncu_winners.py run gpurun_out/r2f_win_$F.json > gpurun_out/r2f_ncu_$F.log 2>&1
done
ls -la gpurun_out/r2f_*
