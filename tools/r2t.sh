timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/r2t_kern.log 2>&1; echo kern_rc=$?
timeout 120 python tools/conv_probe.py fprop 256 13 384 3 1 1 384 20 > gpurun_out/r2t_conv4.log 2>&1
timeout 120 python tools/conv_probe.py fprop 256 27 96 5 1 2 256 20 >> gpurun_out/r2t_conv4.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --profile-out gpurun_out/r2t_prof.json > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; echo bench_rc=$?
