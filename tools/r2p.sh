for d in 0 1 2 4 3 7; do echo "debug=$d"; OMNI_WINDOW_DEBUG=$d timeout 120 python tools/window_probe.py --reps 20 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['window_fprop'])"; done > gpurun_out/r2p_window_debug.log 2>&1
echo done
