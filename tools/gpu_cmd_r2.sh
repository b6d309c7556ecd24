timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -x -p no:cacheprovider -k "tc_every_schedule or split_k or global_splitk or timed_launches" > gpurun_out/r2_red_t.log 2>&1; tail -3 gpurun_out/r2_red_t.log
python tools/gap_trace.py profiles/r02_bench_first.json r50.l3.b0.c2,r50.l3.b1.c1,r50.l3.b1.c2,r50.l4.b0.c2,r50.l4.b1.c1,r50.l4.b1.c2 > gpurun_out/r2_red_gap.log 2>&1
TP_RED_ARRIVE=0 python tools/gap_trace.py profiles/r02_bench_first.json r50.l3.b0.c2,r50.l3.b1.c1,r50.l3.b1.c2,r50.l4.b0.c2,r50.l4.b1.c1,r50.l4.b1.c2 > gpurun_out/r2_red_gap0.log 2>&1
grep -E "^r50|epilogue" gpurun_out/r2_red_gap.log gpurun_out/r2_red_gap0.log
