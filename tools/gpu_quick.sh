timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_schedule" 2>&1 | tail -2
FRAC=0.25 timeout 1200 python tools/explore.py vgg19_b16 vgg.64.224.1,vgg.128.112.0,vgg.128.112.1 gpurun_out/ex_row.json 2>&1 | grep "==" | cut -c1-200
