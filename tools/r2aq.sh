# space-to-depth, one thread per output float4: exact tests + probe A/B.
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "space_to_depth" > gpurun_out/r2aq_tests.log 2>&1; echo tests_rc=$?
timeout 120 python tools/s2d_probe.py > gpurun_out/r2aq_s2d_flat.json 2>&1; echo a=$?
OMNI_S2D_ROWS=1 timeout 120 python tools/s2d_probe.py > gpurun_out/r2aq_s2d_rows.json 2>&1; echo b=$?
