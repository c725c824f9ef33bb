# Streamed 3x3/2 max-pool kernels: parity tests, probe (new vs OMNI_POOL_POINT=1), bench.
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_bench_parity_gpu.py -q -k "pool" > gpurun_out/r2z_tests.log 2>&1; echo tests_rc=$?
timeout 300 python tools/pool_probe.py > gpurun_out/r2z_pool_new.json 2>&1; echo new_rc=$?
OMNI_POOL_POINT=1 timeout 300 python tools/pool_probe.py > gpurun_out/r2z_pool_old.json 2>&1; echo old_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err; echo bench_rc=$?
OMNI_POOL_POINT=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2z_bench_old.json 2> gpurun_out/r2z_bench_old.err; echo bench_old_rc=$?
