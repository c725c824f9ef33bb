# Pool writes the next FC layer's flattened input (no forward transpose): full GPU suite, bench A/B.
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2aw_pytest.log 2>&1; echo pytest_rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2aw_bench_flat$i.json 2> /dev/null; echo flat_rc=$?
OMNI_NO_POOL_FLAT=1 timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2aw_bench_noflat$i.json 2> /dev/null; echo noflat_rc=$?
done
