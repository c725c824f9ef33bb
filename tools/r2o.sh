timeout 2400 python tools/algorithm1_acceptance.py gpurun_out/r2o_algorithm1_acceptance.json > gpurun_out/r2o_a1.log 2>&1; echo a1_rc=$?
