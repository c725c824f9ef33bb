mkdir -p gpurun_out
L=paper_1606_04487_b200/libomni.so
cp $L cur_libomni.so
for r in 1 2; do
 for v in cur alt; do
  cp ${v}_libomni.so $L
  timeout 200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_$v$r.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v$r.json').read().strip().splitlines()[-1]);print('$v',$r,round(d['value']),d['ms_per_step'],d['clocks']['sm_mhz'],d['clocks']['reasons'])"
 done
done
cp cur_libomni.so $L
