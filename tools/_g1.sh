cd /root/repo
timeout 600 python bench.py --steps 3 --warmup 1 --no-extras --no-cpu --no-e2e > gpurun_out/b_ab0.json 2> gpurun_out/b_ab0.err
