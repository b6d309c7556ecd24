#!/bin/bash
# bench line + ncu evidence (launch list, one full capture of the top tensor-core kernel) + reports.
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_r50.py gpurun_out/bench.json 3 > gpurun_out/ncu_launch.log 2>&1
TOP=${TOP_LAYER:-r50.l3.b1.c2}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:igemm -s 2 -c 1 -o gpurun_out/igemm_full python tools/profile_r50.py gpurun_out/bench.json 3 $TOP > gpurun_out/ncu_full.log 2>&1
timeout 1500 python tools/report.py crosseval gpurun_out/r01_crosseval_r50.json > gpurun_out/crosseval.log 2>&1
timeout 1800 python tools/report.py concurrent gpurun_out/r01_concurrent_vgg19.json > gpurun_out/concurrent.log 2>&1
ls -la gpurun_out
