for dbg in 0 32 64; do
 TP_DEBUG_TC=$dbg python tools/tma_probe.py r50.l3.b1.c2 128 32 128 3 256 1
 TP_DEBUG_TC=$dbg python tools/tma_probe.py r50.l4.b1.c1 64 32 128 4 256 1
 TP_DEBUG_TC=$dbg python tools/tma_probe.py r50.l3.b1.c2 128 128 64 4 256 1
done
