cd /root/repo
timeout 900 python -m pytest tests -m gpu -x -q -k "stem" > gpurun_out/st_pytest.log 2>&1
tail -1 gpurun_out/st_pytest.log
for k in 1 2; do timeout 300 python tools/stem_probe.py 2>&1; done
