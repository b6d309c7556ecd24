python tools/trace_sched.py resnet50 r50.conv1 64 32 32 3 256 1 2>&1
python tools/trace_sched.py vgg19_b16 vgg.64.224.0 128 64 16 2 128 1 0.25 2>&1
