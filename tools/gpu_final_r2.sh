#!/bin/bash
# Round-2 evidence in one gpurun call: GPU tests, the bench line, ncu launch list of one bench
# step, per-layer DRAM traffic of the tuned ResNet-50 winners, full captures of the stem and
# resident-weight row kernels at 25%, traces and per-kind probes.
cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest.log
timeout 1200 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?" >> gpurun_out/f_bench.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"igemm|direct" --csv --log-file gpurun_out/f_dram_r50.csv python tools/profile_r50.py gpurun_out/f_bench.json 1 > gpurun_out/f_ncu_dram.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/f_launches_bench.csv python bench.py --profile-steps 1 --warmup 0 > gpurun_out/f_ncu_bench.log 2>&1
FRAC=0.25 KIND=6 TPC=16 timeout 300 ncu --set full --import-source on --clock-control none -k regex:igemm_stem -s 2 -c 1 -o gpurun_out/f_stem_vgg25 -f python tools/run_sched.py vgg19_b16 vgg.64.224.0 128 64 64 2 256 1 > gpurun_out/f_ncu_stem.log 2>&1
FRAC=0.25 KIND=8 TPC=16 timeout 300 ncu --set full --import-source on --clock-control none -k regex:igemm_mt -s 2 -c 1 -o gpurun_out/f_roww_vgg25 -f python tools/run_sched.py vgg19_b16 vgg.64.224.1 128 64 64 6 256 1 > gpurun_out/f_ncu_roww.log 2>&1
timeout 600 python tools/gap_trace.py gpurun_out/f_bench.json > gpurun_out/f_gap.log 2>&1
timeout 300 python tools/stem_probe.py > gpurun_out/f_stem_probe.log 2>&1
timeout 900 python tools/vgg_probe.py 0.25 > gpurun_out/f_vgg_probe.log 2>&1
ls -la gpurun_out | grep " f_"
