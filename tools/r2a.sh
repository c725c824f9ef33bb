set -x
nproc; lscpu | grep "Model name"; free -g | head -2
timeout 1500 python -m pytest tests/test_bench_parity_gpu.py -q -s --durations=0 > gpurun_out/r2a_parity.log 2>&1; echo parity_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err; echo ref_rc=$?
