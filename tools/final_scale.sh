mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multigpu.py -m gpu -x -q > gpurun_out/r01_final_multigpu_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/r01_final_multigpu_pytest.log
timeout 300 python bench.py --gpus 1 > gpurun_out/r01_final_scale_n1.json 2> gpurun_out/r01_final_scale_n1.err
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/r01_final_scale_n$n.json 2> gpurun_out/r01_final_scale_n$n.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/r01_final_ref_n4.json 2> gpurun_out/r01_final_ref_n4.err
tail -2 gpurun_out/r01_final_multigpu_pytest.log
for n in 1 2 4; do python -c "import json,sys;d=json.loads(open('gpurun_out/r01_final_scale_n$n.json').read().strip().splitlines()[-1]);print($n,d['value'],d['e2e']['value'],d['clocks'])"; done
