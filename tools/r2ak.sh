# Momentum-update grid cap (the update stream overlaps the conv backward): bench A/B.
for i in 1 2; do
for cap in 0 148 64 32; do
OMNI_SGD_GRID=$cap timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2ak_bench_cap${cap}_$i.json 2> /dev/null; echo cap${cap}_rc=$?
done
done
