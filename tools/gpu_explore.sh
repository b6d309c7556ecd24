mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; tail -3 gpurun_out/parity.log
timeout 900 python tools/explore.py resnet50 r50.l1.b0.c2,r50.l3.b1.c1,r50.l3.b1.c2,r50.l4.b1.c1,r50.l4.b1.c2,r50.l4.b0.c2 gpurun_out/explore2.json > gpurun_out/explore2.log 2>&1
