# FC bias row, fixed staging pitch: the full GPU suite again.
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2au_pytest.log 2>&1; echo pytest_rc=$?
