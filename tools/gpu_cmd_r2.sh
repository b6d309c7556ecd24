for i in 1 2; do
(cd scratch/r1 && python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > ../../gpurun_out/r2_abr1_$i.json 2>&1)
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extras > gpurun_out/r2_abcur_$i.json 2>&1
done
