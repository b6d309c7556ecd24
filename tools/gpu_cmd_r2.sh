timeout 900 python -m pytest tests/test_gpu_r2.py -q --timeout 600 -p no:cacheprovider -k "strip" > gpurun_out/r2_strip_t5.log 2>&1; tail -2 gpurun_out/r2_strip_t5.log
timeout 900 python tools/vgg_probe.py 0.25 vgg.64.224.0 > gpurun_out/r2_vgg_probe5.log 2>&1; cat gpurun_out/r2_vgg_probe5.log
python tools/mt_trace.py vgg19_b16 vgg.64.224.0 166 0.25 > gpurun_out/r2_mt_trace2.log 2>&1; cat gpurun_out/r2_mt_trace2.log
