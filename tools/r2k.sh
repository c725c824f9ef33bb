export NCCL_DEBUG=WARN
for g in 1 2; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tests/mp_async_check.py cifar10_quick $g 16 > gpurun_out/r2k_async_g$g.log 2>&1; echo async_g$g=$?; done
timeout 900 python -m pytest tests/test_multigpu.py -q > gpurun_out/r2k_multigpu.log 2>&1; echo multigpu_rc=$?
