timeout 120 ./tools/mma_probe > gpurun_out/r2e_mma.log 2>&1; echo mma_rc=$?
timeout 300 python tools/window_probe.py > gpurun_out/r2e_probe.json 2> gpurun_out/r2e_probe.err; echo probe_rc=$?
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q > gpurun_out/r2e_kern.log 2>&1; echo kern_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --profile-out gpurun_out/r2e_prof.json > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo bench_rc=$?
