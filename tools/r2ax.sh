# Clock sampling inside the timed region (sampler waits for its first sample).
timeout 600 python bench.py > gpurun_out/r2ax_bench.json 2> gpurun_out/r2ax_bench.err; echo bench_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29641 bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ax_torchrun.json 2> gpurun_out/r2ax_torchrun.err; echo tr_rc=$?
