# Pool kernels incl. the engine's marked form; ncu of the marked stride-2 backward (pool1).
timeout 300 python tools/pool_probe.py > gpurun_out/r2am_pool.json 2>&1; echo probe_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_bwd -s 1 -c 1 -o gpurun_out/r2am_poolbwd python tools/pool_probe.py --once > gpurun_out/r2am_ncu.log 2>&1; echo ncu_rc=$?
