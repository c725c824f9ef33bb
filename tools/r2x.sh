# 4-GPU: the co-located async group checks (N=4, g=2 failed once in r2_scale) with full tracebacks.
export NCCL_DEBUG=WARN
for i in 1 2; do timeout 900 python -m pytest tests/test_multigpu.py -q -k "colocated" > gpurun_out/r2x_coloc_$i.log 2>&1; echo coloc${i}_rc=$?; done
for g in 2; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2971$g tests/mp_async_check.py cifar10_quick $g 16 > gpurun_out/r2x_check_g$g.log 2>&1; echo check_g${g}=$?; done
