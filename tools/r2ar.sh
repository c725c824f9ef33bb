# GroupRuntime.close on GPUs: the group-runtime multi-GPU tests and a groups bench at N=2.
export NCCL_DEBUG=WARN
timeout 1200 python -m pytest tests/test_multigpu.py -q -k "group_runtime" > gpurun_out/r2ar_tests.log 2>&1; echo tests_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 10 --warmup 3 --groups 2 > gpurun_out/r2ar_g2.json 2> gpurun_out/r2ar_g2.err; echo g2_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 --steps 10 --warmup 3 --groups 2 --groups-nccl > gpurun_out/r2ar_g2n.json 2> gpurun_out/r2ar_g2n.err; echo g2n_rc=$?
