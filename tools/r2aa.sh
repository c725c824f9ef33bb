# Max-pool kernels with every window load issued up front: parity tests, probe, bench.
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_bench_parity_gpu.py -q -k "pool" > gpurun_out/r2aa_tests.log 2>&1; echo tests_rc=$?
timeout 300 python tools/pool_probe.py > gpurun_out/r2aa_pool.json 2>&1; echo probe_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --profile-out gpurun_out/r2aa_prof.json > gpurun_out/r2aa_bench.json 2> gpurun_out/r2aa_bench.err; echo bench_rc=$?
git_stash_note="(no A/B arm: the previous kernels' numbers are r2z_pool_old.json / profiles/r02_pool_streamed_ab.json)"
