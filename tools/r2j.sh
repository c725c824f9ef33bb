timeout 1500 ncu --nvtx --nvtx-include "step/" --set full --clock-control none -o /tmp/r2j_step python tools/profile_step.py caffenet 256 > gpurun_out/r2j_ncu.log 2>&1; echo ncu_rc=$?
ncu -i /tmp/r2j_step.ncu-rep --page raw --csv > gpurun_out/r2j_step_raw.csv 2>/dev/null; echo raw_rc=$?
ls -la /tmp/r2j_step.ncu-rep gpurun_out/r2j_step_raw.csv
