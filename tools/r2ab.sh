# Staged space-to-depth: kernel tests, probe (staged vs OMNI_S2D_V4=1), bench A/B on one box.
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "space_to_depth or window or s2d" > gpurun_out/r2ab_tests.log 2>&1; echo tests_rc=$?
cat > /tmp/s2d_probe.py <<'PY'
import json, sys, torch
sys.path.insert(0, '.')
from paper_1606_04487_b200 import kernels as K
b, n, c, s = 256, 227, 3, 4
X = torch.randn(b, n, n, c, device='cuda'); idx = torch.randperm(b, device='cuda')
Y = torch.empty(b, 57, 57, 48, device='cuda')
K.space_to_depth_gather(X, idx, c, s, Y); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): K.space_to_depth_gather(X, idx, c, s, Y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
nb = 4 * b * n * n * c + 4 * b * 57 * 57 * 48
print(json.dumps({"us": ms * 1e3, "GBps": nb / ms / 1e6}))
PY
timeout 120 python /tmp/s2d_probe.py > gpurun_out/r2ab_s2d_staged.json 2>&1; echo s2d_rc=$?
OMNI_S2D_V4=1 timeout 120 python /tmp/s2d_probe.py > gpurun_out/r2ab_s2d_v4.json 2>&1; echo s2d4_rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2ab_bench_new$i.json 2> gpurun_out/r2ab_bench_new$i.err; echo bench_new_rc=$?
OMNI_S2D_V4=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2ab_bench_v4_$i.json 2> gpurun_out/r2ab_bench_v4_$i.err; echo bench_v4_rc=$?
done
