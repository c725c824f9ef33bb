timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "window" > gpurun_out/r2h_window.log 2>&1; echo window_rc=$?
timeout 300 python tools/window_probe.py > gpurun_out/r2h_probe.json 2> gpurun_out/r2h_probe.err; echo probe_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_window -c 3 -o gpurun_out/r2h_window python tools/window_probe.py --once > gpurun_out/r2h_ncu.log 2>&1; echo ncu_rc=$?
