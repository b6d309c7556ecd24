#!/bin/bash
# Round evidence: GPU tests, bench line, ncu (launch list of one bench step, per-layer DRAM traffic of
# the tuned R50 schedules, full capture of the top kernel), experiment reports.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:igemm --csv --log-file gpurun_out/dram_r50.csv python tools/profile_r50.py gpurun_out/bench.json 1 > gpurun_out/ncu_dram.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --profile-steps 1 --warmup 0 > gpurun_out/ncu_bench.log 2>&1
TOP=${TOP_LAYER:-r50.l3.b1.c2}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:igemm -s 2 -c 1 -o gpurun_out/igemm_full python tools/profile_r50.py gpurun_out/bench.json 3 $TOP > gpurun_out/ncu_full.log 2>&1
timeout 1500 python tools/report.py crosseval gpurun_out/r01_crosseval_r50.json > gpurun_out/crosseval.log 2>&1
timeout 1800 python tools/report.py concurrent gpurun_out/r01_concurrent_vgg19.json > gpurun_out/concurrent.log 2>&1
timeout 900 python tools/report.py tune gpurun_out/r01_tune_mbv2_50.json > gpurun_out/mbv2.log 2>&1
ls -la gpurun_out | tail -20
timeout 600 python tools/report.py tune --workload cfg1 --fraction 1.0 gpurun_out/r01_tune_cfg1_100.json > gpurun_out/cfg1.log 2>&1
timeout 1200 python tools/report.py interference gpurun_out/r01_interference_r50.json > gpurun_out/interference.log 2>&1
