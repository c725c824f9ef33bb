timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "window" > gpurun_out/r2c_window.log 2>&1; echo window_rc=$?
timeout 900 python -m pytest tests/ -q -x -m gpu --ignore=tests/test_bench_parity_gpu.py > gpurun_out/r2c_gpu.log 2>&1; echo gpu_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --profile-out gpurun_out/r2c_prof.json > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo bench_rc=$?
timeout 600 python -m pytest tests/test_bench_parity_gpu.py -q -s -k "layer_isolated and tf32" > gpurun_out/r2c_parity.log 2>&1; echo parity_rc=$?
