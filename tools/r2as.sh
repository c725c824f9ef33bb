# Split-K reduce with 4 split loads in flight: GEMM tests, bench, launch list.
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "gemm" > gpurun_out/r2as_tests.log 2>&1; echo tests_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2as_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2as_ncu.log 2>&1; echo ncu_rc=$?
