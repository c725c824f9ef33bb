# ncu --set full of every launch of one eager CaffeNet step with the final kernels.
timeout 1800 ncu --nvtx --nvtx-include "step/" --set full --clock-control none -o /tmp/r2ao_step python tools/profile_step.py caffenet 256 > gpurun_out/r2ao_ncu.log 2>&1; echo ncu_rc=$?
ncu -i /tmp/r2ao_step.ncu-rep --page raw --csv > gpurun_out/r2ao_step_raw.csv 2>/dev/null; echo raw_rc=$?
ls -la gpurun_out/r2ao_step_raw.csv
