timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "window" > gpurun_out/r2q_window.log 2>&1; echo window_rc=$?
for d in 0 1 3; do echo "debug=$d"; OMNI_WINDOW_DEBUG=$d timeout 120 python tools/window_probe.py --reps 20 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['window_fprop'])"; done > gpurun_out/r2q_window_debug.log 2>&1
timeout 2400 python tools/algorithm1_acceptance.py gpurun_out/r2q_algorithm1_acceptance.json > gpurun_out/r2q_a1.log 2>&1; echo a1_rc=$?
