timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tuner.py -x -q 2>&1 | tail -3
python tools/trace_sched.py resnet50 r50.conv1 64 32 32 3 256 1
python tools/trace_sched.py resnet50 r50.conv1 128 64 64 3 256 1
python tools/trace_sched.py vgg19_b16 vgg.64.224.0 128 64 16 2 128 1 0.25
python tools/trace_sched.py vgg19_b16 vgg.64.224.0 128 64 32 2 256 1 0.25
