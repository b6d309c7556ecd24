cd /root/repo
timeout 300 python tools/stem_probe.py > gpurun_out/st_probe_1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gather or stem" > gpurun_out/st_pytest.log 2>&1
tail -1 gpurun_out/st_pytest.log
