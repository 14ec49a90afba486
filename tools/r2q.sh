timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2q_pytest.log 2>&1; tail -3 gpurun_out/r2q_pytest.log
timeout 300 python tools/profile_e.py 2 2>&1 | tail -1
timeout 300 python tools/batch_probe.py B 2>&1 | grep -E '"batch": (1|8)'
