# conv1 weight-gradient reduction with 8 lanes per output: tests, probe, launch list.
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "window" > gpurun_out/r2ap_tests.log 2>&1; echo tests_rc=$?
timeout 1200 python -m pytest tests/test_bench_parity_gpu.py -q -k "isolated and tf32 and not 3x" > gpurun_out/r2ap_parity.log 2>&1; echo parity_rc=$?
timeout 300 python tools/window_probe.py > gpurun_out/r2ap_probe.json 2>&1; echo probe_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:window -c 20 --csv --log-file gpurun_out/r2ap_launches.csv python tools/window_probe.py --once > gpurun_out/r2ap_ncu.log 2>&1; echo ncu_rc=$?
