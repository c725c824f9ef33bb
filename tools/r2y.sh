# Pooling kernels alone (CaffeNet b=256) + one ncu --set full capture of pool1 forward and backward.
timeout 300 python tools/pool_probe.py > gpurun_out/r2y_pool.json 2>&1; echo pool_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool -c 2 -o gpurun_out/r2y_pool python tools/pool_probe.py --once > gpurun_out/r2y_ncu.log 2>&1; echo ncu_rc=$?
