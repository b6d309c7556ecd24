timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_schedule" 2>&1 | tail -2
for L in vgg.64.224.1 vgg.128.112.0; do
FRAC=0.25 timeout 600 python tools/explore.py vgg19_b16 $L gpurun_out/ex_b.json 2>&1 | grep "=="
TP_NO_BRES=1 FRAC=0.25 timeout 600 python tools/explore.py vgg19_b16 $L gpurun_out/ex_nb.json 2>&1 | grep "=="
done
