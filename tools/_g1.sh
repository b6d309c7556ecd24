cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q -k "row or roww or strip or mt" > gpurun_out/st_pytest.log 2>&1
tail -1 gpurun_out/st_pytest.log
timeout 600 python tools/vgg_probe.py 0.25 vgg.64.224.1,vgg.128.112.0 > gpurun_out/vgg_probe.log 2>&1
TP_MMA2=0 timeout 600 python tools/vgg_probe.py 0.25 vgg.64.224.1,vgg.128.112.0 > gpurun_out/vgg_probe0.log 2>&1
