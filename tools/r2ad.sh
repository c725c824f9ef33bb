# ncu --set full of the max-pool backward (pool1 shape) after the up-front-loads change.
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_bwd -c 1 -o gpurun_out/r2ad_poolbwd python tools/pool_probe.py --once > gpurun_out/r2ad_ncu.log 2>&1; echo ncu_rc=$?
