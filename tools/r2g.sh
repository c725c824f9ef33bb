timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_window -c 3 -o gpurun_out/r2g_window python tools/window_probe.py --once > gpurun_out/r2g_ncu.log 2>&1; echo ncu_rc=$?
