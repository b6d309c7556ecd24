cd /root/repo
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "stem" > gpurun_out/st_pytest.log 2>&1
tail -1 gpurun_out/st_pytest.log
timeout 300 python tools/stem_probe.py > gpurun_out/st_probe_1.log 2>&1
