cd /root/repo
timeout 600 python tools/gap_trace.py profiles/r02_bench.json r50.l1.b0.c1,r50.l2.b0.c2,r50.l3.b0.c2,r50.l4.b0.c1 > gpurun_out/gap.log 2>&1
