timeout 900 python tools/algorithm1_calibrate.py > gpurun_out/r2m_calib.log 2>&1; echo calib_rc=$?
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/r2m_memcheck.log 2>&1; echo memcheck_rc=$?
