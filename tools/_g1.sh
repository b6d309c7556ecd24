cd /root/repo
timeout 1200 python -m pytest tests -m gpu -x -q -k "row or strip or mt or stem or roww or tma_store" > gpurun_out/st_pytest.log 2>&1
tail -3 gpurun_out/st_pytest.log
timeout 600 python tools/vgg_probe.py 0.25 vgg.64.224.0,vgg.64.224.1,vgg.128.112.0,vgg.128.112.1 > gpurun_out/vgg_probe.log 2>&1
