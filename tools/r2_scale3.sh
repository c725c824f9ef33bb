# Round-2 multi-GPU validation (gpurun --gpus 4): multi-GPU parity tests, the
# C-ABI collectives check, DP scaling N=1,2,4, and the compute-group runtime
# (peer-memory and NCCL-sharded rounds) at N=4.
export NCCL_DEBUG=WARN
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 1500 python -m pytest tests/test_multigpu.py "tests/test_kernels_gpu.py::test_group_updates_equals_eager_rounds" -q -m gpu > gpurun_out/scale3_pytest.log 2>&1; echo pytest_rc=$?
run 4 29601 tools/comm_check.py > gpurun_out/scale3_comm_check.log 2>&1; echo comm_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/scale3_n1.json 2> gpurun_out/scale3_n1.err; echo n1_rc=$?
run 2 29602 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/scale3_n2.json 2> gpurun_out/scale3_n2.err; echo n2_rc=$?
run 4 29604 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/scale3_n4.json 2> gpurun_out/scale3_n4.err; echo n4_rc=$?
for g in 2 4; do run 4 2961$g bench.py --gpus 4 --steps 20 --warmup 5 --groups $g > gpurun_out/scale3_n4_g$g.json 2> gpurun_out/scale3_n4_g$g.err; echo g${g}_rc=$?; done
run 4 29620 bench.py --gpus 4 --steps 20 --warmup 5 --groups 2 --groups-nccl > gpurun_out/scale3_n4_g2_nccl.json 2> gpurun_out/scale3_n4_g2_nccl.err; echo g2nccl_rc=$?
run 4 29621 bench.py --gpus 4 --steps 20 --warmup 5 --groups 2 --groups-nccl --groups-overlap > gpurun_out/scale3_n4_g2_nccl_ovl.json 2> gpurun_out/scale3_n4_g2_nccl_ovl.err; echo g2ovl_rc=$?
