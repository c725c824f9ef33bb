# FC bias gradient as one more row of the weight-gradient GEMM: full GPU suite, bench A/B, launch list.
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2at_pytest.log 2>&1; echo pytest_rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2at_bench_row$i.json 2> /dev/null; echo row_rc=$?
OMNI_NO_FC_BIAS_ROW=1 timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2at_bench_norow$i.json 2> /dev/null; echo norow_rc=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2at_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2at_ncu.log 2>&1; echo ncu_rc=$?
