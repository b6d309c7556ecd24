cd /root/repo
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tuner.py -m gpu -x -q > gpurun_out/st_pytest.log 2>&1
tail -1 gpurun_out/st_pytest.log
timeout 900 python bench.py --steps 3 --warmup 1 --no-extras --no-cpu --no-e2e > gpurun_out/b_ab.json 2> gpurun_out/b_ab.err
