cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q -k "stem or row or strip or mt or roww or tma_store" > gpurun_out/st_pytest.log 2>&1
tail -1 gpurun_out/st_pytest.log
timeout 300 python tools/stem_probe.py > gpurun_out/st_probe_1.log 2>&1
timeout 600 python tools/vgg_probe.py 0.25 vgg.64.224.1,vgg.128.112.0 > gpurun_out/vgg_probe.log 2>&1
