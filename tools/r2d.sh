timeout 300 python tools/window_probe.py > gpurun_out/r2d_probe.json 2> gpurun_out/r2d_probe.err; echo probe_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_window -c 3 -o gpurun_out/r2d_window python tools/window_probe.py --once > gpurun_out/r2d_ncu.log 2>&1; echo ncu_rc=$?
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/r2d_kern.log 2>&1; echo kern_rc=$?
