timeout 60 ./tools/desc_probe > gpurun_out/r2b_probe.log 2>&1; echo probe_rc=$?
timeout 1500 python -m pytest tests/test_bench_parity_gpu.py -q -s > gpurun_out/r2b_parity.log 2>&1; echo parity_rc=$?
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_kernels_gpu.py -q -x > gpurun_out/r2b_kern.log 2>&1; echo kern_rc=$?
