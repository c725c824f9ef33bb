# Window wgrad v2 (ring of s2d rows, M = (kx, ky*48+ch)): kernel tests, isolated
# timing vs the generic implicit wgrad, bench, ncu of the new kernel.
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "window or group_updates or partial_channel" > gpurun_out/r2w_kern.log 2>&1; echo kern_rc=$?
timeout 300 python tools/window_probe.py > gpurun_out/r2w_probe.json 2>&1; echo probe_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --profile-out gpurun_out/r2w_prof.json > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err; echo bench_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_window_wgrad -c 1 -o gpurun_out/r2w_wgrad python tools/window_probe.py --once > gpurun_out/r2w_ncu.log 2>&1; echo ncu_rc=$?
