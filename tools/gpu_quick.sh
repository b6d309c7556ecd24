timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 600 python tools/explore.py resnet50 r50.conv1 gpurun_out/ex_pad_r50.json 2>&1 | grep "=="
FRAC=0.25 timeout 900 python tools/explore.py vgg19_b16 vgg.64.224.0 gpurun_out/ex_pad_vgg.json 2>&1 | grep "=="
