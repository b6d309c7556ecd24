timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider -k "strip or multitile or ytma_mt or slots or row" > gpurun_out/r2_epi_t.log 2>&1; tail -4 gpurun_out/r2_epi_t.log
timeout 900 python tools/vgg_probe.py 0.25 > gpurun_out/r2_vgg_probe_ys2.log 2>&1; cat gpurun_out/r2_vgg_probe_ys2.log
TP_YSTAGE2=0 timeout 900 python tools/vgg_probe.py 0.25 vgg.64.224.0,vgg.64.224.1,vgg.128.112.0,vgg.128.112.1 > gpurun_out/r2_vgg_probe_ys1.log 2>&1; cat gpurun_out/r2_vgg_probe_ys1.log
