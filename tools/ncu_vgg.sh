#!/bin/bash
# ncu (tensor pipe, DRAM, duration; cold caches) of every VGG-19 b16 winner of the concurrent-tuner report, run in a 25% partition
mkdir -p gpurun_out
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.sum,sm__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size
for L in vgg.64.224.0 vgg.64.224.1 vgg.128.112.0 vgg.128.112.1 vgg.256.56.0 vgg.256.56.1 vgg.512.28.0 vgg.512.28.1 vgg.512.14.0; do
  IDX=$(python -c "import json; d=json.load(open('profiles/r01_concurrent_vgg19.json')); print([r for r in d['layers'] if r['layer']=='$L'][0]['schedule']['space_index'])")
  FRAC=0.25 timeout 300 ncu --metrics $M --clock-control none -k regex:"igemm|stem" -s 2 -c 1 --csv --log-file gpurun_out/ncuf_${L}_0.25.csv python tools/run_idx.py vgg19_b16 $L $IDX 3 > /dev/null 2>&1
done
ls gpurun_out/ncuf_vgg* | wc -l
