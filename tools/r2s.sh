timeout 120 python tools/conv_probe.py fprop 256 13 384 3 1 1 384 20 > gpurun_out/r2s_conv4.log 2>&1
OMNI_FORCE_BN=128 timeout 120 python tools/conv_probe.py fprop 256 13 384 3 1 1 384 20 >> gpurun_out/r2s_conv4.log 2>&1
OMNI_FORCE_BN=256 timeout 120 python tools/conv_probe.py fprop 256 13 384 3 1 1 384 20 >> gpurun_out/r2s_conv4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -c 1 -s 2 -o gpurun_out/r2s_conv4 python tools/conv_probe.py fprop 256 13 384 3 1 1 384 1 > gpurun_out/r2s_ncu.log 2>&1; echo ncu_rc=$?
