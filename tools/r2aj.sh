# Default build with 3xTF32 pairs on plain GEMMs: kernel tests (both precisions), parity, probe timing.
timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q > gpurun_out/r2aj_tests.log 2>&1; echo tests_rc=$?
timeout 300 python tools/x3pair_probe.py --timing > gpurun_out/r2aj_time.json 2>&1; echo t_rc=$?
