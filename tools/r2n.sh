export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_multigpu.py -q -k "data_parallel" > gpurun_out/r2n_multigpu.log 2>&1; echo multigpu_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --steps 20 --warmup 5 --nccl-allreduce > gpurun_out/r2n_dp_nccl_n2.json 2> gpurun_out/r2n_dp_nccl_n2.err; echo nccl_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --steps 20 --warmup 5 --merged-fc > gpurun_out/r2n_mergedfc_n2.json 2> gpurun_out/r2n_mergedfc_n2.err; echo merged_rc=$?
