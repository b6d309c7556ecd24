python tools/gap_trace.py profiles/r02_bench_first.json r50.l1.b0.c1,r50.l1.b0.c3,r50.l3.b0.c3 > gpurun_out/r2_gap5a.log 2>&1
TP_DEBUG_TC=4 python tools/gap_trace.py profiles/r02_bench_first.json r50.l1.b0.c1,r50.l1.b0.c3,r50.l3.b0.c3 > gpurun_out/r2_gap5b.log 2>&1
