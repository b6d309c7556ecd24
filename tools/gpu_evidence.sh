#!/bin/bash
# Trace of the gathered stem + ncu evidence: per-layer DRAM traffic of the tuned R50 schedules,
# launch list of one bench step, full captures at 25% (VGG, tensor-bound) and 50% (MBv2 dw, HBM-bound).
mkdir -p gpurun_out
python tools/trace_sched.py resnet50 r50.conv1 64 32 32 3 256 1 > gpurun_out/tr_gather.log 2>&1
python tools/trace_sched.py vgg19_b16 vgg.64.224.0 128 64 16 2 128 1 0.25 >> gpurun_out/tr_gather.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:igemm --csv --log-file gpurun_out/dram_r50.csv python tools/profile_r50.py profiles/r01_bench.json 1 > gpurun_out/ncu_dram.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --profile-steps 1 --warmup 0 > gpurun_out/ncu_bench.log 2>&1
FRAC=0.25 timeout 600 ncu --set full --clock-control none --import-source on -k regex:igemm -s 1 -c 1 -o gpurun_out/vgg_512_28_1_p25 python tools/run_sched.py vgg19_b16 vgg.512.28.1 128 256 64 2 128 1 2 > gpurun_out/ncu_vgg.log 2>&1
FRAC=0.5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:direct -s 1 -c 1 -o gpurun_out/mb2_dw_p50 python tools/run_sched.py mobilenetv2 mb2.dw.96.112.s2 D 256 2 8 2 0 2 > gpurun_out/ncu_mb2.log 2>&1
ls -la gpurun_out | tail -12
