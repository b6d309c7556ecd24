mkdir -p gpurun_out
timeout 1800 python tools/report.py concurrent gpurun_out/r01_concurrent_vgg19.json > gpurun_out/concurrent.log 2>&1
