# ncu --set full of the conv1 window forward kernel alone (b=256).
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_window_fprop -c 1 -o gpurun_out/r2ag_fprop python tools/window_probe.py --once > gpurun_out/r2ag_ncu.log 2>&1; echo ncu_rc=$?
