timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "window" > gpurun_out/r2r_window.log 2>&1; echo window_rc=$?
for d in 0 1; do echo "debug=$d"; OMNI_WINDOW_DEBUG=$d timeout 120 python tools/window_probe.py --reps 20 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['window_fprop'])"; done > gpurun_out/r2r_window_debug.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --profile-out gpurun_out/r2r_prof.json > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; echo bench_rc=$?
