timeout 300 python tools/x3pair_probe.py > gpurun_out/r2ah_single.json 2>&1; echo single_rc=$?
OMNI_3X_PAIRS=1 timeout 300 python tools/x3pair_probe.py > gpurun_out/r2ah_pairs.json 2>&1; echo pairs_rc=$?
