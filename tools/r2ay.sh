# Variance of the NCCL sharded group rounds at N=4, g=2 (three runs).
export NCCL_DEBUG=WARN
for i in 1 2 3; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2965$i bench.py --gpus 4 --steps 20 --warmup 5 --groups 2 --groups-nccl > gpurun_out/r2ay_g2nccl_$i.json 2> /dev/null; echo rc=$?; done
