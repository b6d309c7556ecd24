mkdir -p gpurun_out
for nacc in 1 2 4; do
 TP_NACC=$nacc python tools/tma_probe.py r50.l4.b1.c1 64 32 128 4 256 1
 TP_NACC=$nacc python tools/tma_probe.py r50.l3.b1.c2 128 32 128 3 256 1
 TP_NACC=$nacc python tools/tma_probe.py r50.l3.b1.c2 128 128 64 4 256 1
 TP_NACC=$nacc python tools/tma_probe.py r50.l1.b0.c1 128 32 64 6 256 1
done
TP_DEBUG_TC=3 python tools/tma_probe.py r50.l3.b1.c2 128 32 128 3 256 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
TP_NACC=4 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
