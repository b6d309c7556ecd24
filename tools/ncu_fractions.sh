#!/bin/bash
# ncu of the tuned winner at each SM fraction (cross-eval report schedules): tensor-pipe and DRAM evidence
mkdir -p gpurun_out
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size
for L in r50.l3.b1.c2 r50.l1.b0.c2 r50.conv1; do
  for F in 0.1 0.25 0.5 1.0; do
    IDX=$(python -c "import json; d=json.load(open('profiles/r01_crosseval_r50.json')); print([r for r in d['layers'] if r['layer']=='$L'][0]['best_schedule']['$F']['space_index'])")
    FRAC=$F timeout 300 ncu --metrics $M --clock-control none -k regex:igemm -s 2 -c 1 --csv --log-file gpurun_out/ncuf_${L}_${F}.csv python tools/run_idx.py resnet50 $L $IDX 3 > /dev/null 2>&1
  done
done
for F in 0.25; do
  FRAC=$F timeout 300 ncu --metrics $M --clock-control none -k regex:igemm -s 1 -c 1 --csv --log-file gpurun_out/ncuf_vgg.512.28.1_${F}.csv python tools/run_sched.py vgg19_b16 vgg.512.28.1 128 256 64 2 128 1 2 > /dev/null 2>&1
done
ls gpurun_out/ncuf_* | wc -l
