timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_dropin.py > gpurun_out/r2s_pytest.log 2>&1; tail -3 gpurun_out/r2s_pytest.log
timeout 300 python tools/profile_e.py 2 2>&1 | tail -1
timeout 300 python tools/batch_probe.py B C 2>&1 | grep -E '"batch": (1|8)'
CHECK_ITERS=0 timeout 600 python tools/bench_configs.py 3 A D 2>&1 | tail -2
