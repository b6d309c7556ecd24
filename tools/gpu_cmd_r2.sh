timeout 300 python -m pytest tests/test_gpu_r2.py -q --timeout 120 -x -p no:cacheprovider -k "roww" > gpurun_out/r2_pair_t0.log 2>&1; tail -3 gpurun_out/r2_pair_t0.log
TP_ROWW2=1 timeout 300 python -m pytest tests/test_gpu_r2.py -q --timeout 120 -x -p no:cacheprovider -k "roww" > gpurun_out/r2_pair_t1.log 2>&1; tail -3 gpurun_out/r2_pair_t1.log
TP_ROWW2=1 timeout 600 python tools/vgg_probe.py 0.25 vgg.64.224.1,vgg.128.112.0 > gpurun_out/r2_vgg_probe12.log 2>&1; cat gpurun_out/r2_vgg_probe12.log
timeout 600 python tools/vgg_probe.py 0.25 vgg.64.224.1,vgg.128.112.0 > gpurun_out/r2_vgg_probe12b.log 2>&1; cat gpurun_out/r2_vgg_probe12b.log
