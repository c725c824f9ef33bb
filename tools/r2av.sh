# Pool backward with multiply-shift index division: pool tests, probe.
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_bench_parity_gpu.py -q -k "pool" > gpurun_out/r2av_tests.log 2>&1; echo tests_rc=$?
timeout 300 python tools/pool_probe.py > gpurun_out/r2av_pool.json 2>&1; echo probe_rc=$?
