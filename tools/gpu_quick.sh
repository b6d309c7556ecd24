timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
FRAC=0.25 timeout 1500 python tools/explore.py vgg19_b16 vgg.256.56.0,vgg.256.56.1,vgg.512.28.0,vgg.512.28.1 gpurun_out/ex_mt.json 2>&1 | grep "=="
