# Round-2 final validation on one fresh box: GPU tests, smoke, both bench arms,
# the 3xTF32 line, and the ncu launch list of the bench command.
export NCCL_DEBUG=WARN
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/final6_pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final6_ref.json 2> gpurun_out/final6_ref.err; echo ref_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final6_bench.json 2> gpurun_out/final6_bench.err; echo bench_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --precision 3xtf32 --no-cpu-baseline > gpurun_out/final6_bench_3xtf32.json 2> gpurun_out/final6_bench_3xtf32.err; echo bench3_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/final6_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final6_ncu.log 2>&1; echo ncu_rc=$?
