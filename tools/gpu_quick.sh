timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_schedule" 2>&1 | tail -2
KIND=3 python tools/trace_sched.py vgg19_b16 vgg.64.224.1 128 64 64 1 256 1 0.25
KIND=3 python tools/trace_sched.py vgg19_b16 vgg.64.224.1 128 64 64 1 128 1 0.25
KIND=3 python tools/trace_sched.py vgg19_b16 vgg.128.112.0 128 128 64 1 256 1 0.25
