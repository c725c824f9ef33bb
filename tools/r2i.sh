timeout 900 python -m pytest tests/ -q -m gpu --ignore=tests/test_bench_parity_gpu.py > gpurun_out/r2i_gpu.log 2>&1; echo gpu_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --profile-out gpurun_out/r2i_prof.json > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo bench_rc=$?
timeout 900 python -m pytest tests/test_bench_parity_gpu.py -q -s -k "caffenet" > gpurun_out/r2i_parity.log 2>&1; echo parity_rc=$?
