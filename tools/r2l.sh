export NCCL_DEBUG=WARN
for g in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2952$g tests/mp_async_check.py cifar10_quick $g 24 > gpurun_out/r2l_async_check_g$g.log 2>&1; echo check_g$g=$?; done
for g in 1 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$g tools/async_colocated_bench.py $g 60 256 caffenet > gpurun_out/r2l_async_caffenet_g$g.json 2> gpurun_out/r2l_async_caffenet_g$g.err; echo bench_g$g=$?; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29540 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2l_dp_n4.json 2> gpurun_out/r2l_dp_n4.err; echo dp_rc=$?
