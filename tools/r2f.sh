timeout 120 ./tools/mma_probe > gpurun_out/r2f_mma.log 2>&1; echo mma_rc=$?
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "window" > gpurun_out/r2f_window.log 2>&1; echo window_rc=$?
timeout 300 python tools/window_probe.py > gpurun_out/r2f_probe.json 2> gpurun_out/r2f_probe.err; echo probe_rc=$?
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q > gpurun_out/r2f_kern.log 2>&1; echo kern_rc=$?
