# 3xTF32 on CTA pairs (OMNI_3X_PAIRS=1): numerics vs single CTAs, kernel tests, timing, bench.
timeout 300 python tools/x3pair_probe.py > gpurun_out/r2ai_single.json 2>&1; echo single_rc=$?
OMNI_3X_PAIRS=1 timeout 300 python tools/x3pair_probe.py > gpurun_out/r2ai_pairs.json 2>&1; echo pairs_rc=$?
timeout 300 python tools/x3pair_probe.py --timing > gpurun_out/r2ai_time_single.json 2>&1; echo t1=$?
OMNI_3X_PAIRS=1 timeout 300 python tools/x3pair_probe.py --timing > gpurun_out/r2ai_time_pairs.json 2>&1; echo t2=$?
OMNI_3X_PAIRS=1 timeout 1200 python -m pytest tests/test_kernels_gpu.py -q -k "3xtf32 or 3XTF32 or PREC_3X" > gpurun_out/r2ai_kern.log 2>&1; echo kern_rc=$?
OMNI_3X_PAIRS=1 timeout 1200 python -m pytest tests/test_bench_parity_gpu.py -q -k "isolated and 3x" > gpurun_out/r2ai_parity.log 2>&1; echo parity_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 --precision 3xtf32 --no-cpu-baseline --no-e2e > gpurun_out/r2ai_bench_single.json 2> gpurun_out/r2ai_bench_single.err; echo b1=$?
OMNI_3X_PAIRS=1 timeout 900 python bench.py --steps 10 --warmup 3 --precision 3xtf32 --no-cpu-baseline --no-e2e > gpurun_out/r2ai_bench_pairs.json 2> gpurun_out/r2ai_bench_pairs.err; echo b2=$?
