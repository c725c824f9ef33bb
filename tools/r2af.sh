# Max pools over ReLU outputs with the mask folded into the argmax (forward mode 2):
# kernel tests, the engine-level parity test, bench A/B on one box.
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "pool" > gpurun_out/r2af_tests.log 2>&1; echo tests_rc=$?
timeout 1200 python -m pytest tests/test_bench_parity_gpu.py -q -k "isolated and tf32 and not 3x" > gpurun_out/r2af_parity.log 2>&1; echo parity_rc=$?
timeout 600 python tools/pool_probe.py > gpurun_out/r2af_pool.json 2>&1; echo probe_rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2af_bench_mark$i.json 2> gpurun_out/r2af_bench_mark$i.err; echo mark_rc=$?
OMNI_NO_POOL_MARK=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2af_bench_nomark$i.json 2> gpurun_out/r2af_bench_nomark$i.err; echo nomark_rc=$?
done
