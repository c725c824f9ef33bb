# Co-located async groups at N=4 with the HE check (phase profile measured on the box).
export NCCL_DEBUG=WARN
for g in 1 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2981$g tools/async_colocated_bench.py $g 60 256 caffenet > gpurun_out/r2al_async_g$g.json 2> gpurun_out/r2al_async_g$g.err; echo g${g}_rc=$?; done
