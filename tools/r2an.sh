# space-to-depth with all 16 loads per thread issued up front: exact test + probe.
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "space_to_depth or window" > gpurun_out/r2an_tests.log 2>&1; echo tests_rc=$?
timeout 120 python tools/s2d_probe.py > gpurun_out/r2an_s2d.json 2>&1; echo s2d_rc=$?
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "transpose" > gpurun_out/r2an_transpose.log 2>&1; echo tr_rc=$?
for i in 1 2 3; do timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --profile-out gpurun_out/r2an_prof$i.json > gpurun_out/r2an_bench$i.json 2> /dev/null; echo bench_rc=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2an_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2an_ncu.log 2>&1; echo ncu_rc=$?
