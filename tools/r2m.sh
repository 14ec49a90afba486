timeout 1500 python -m pytest tests/test_dropin.py tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/r2m_dropin.log 2>&1; tail -15 gpurun_out/r2m_dropin.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_parity_configs.py > gpurun_out/r2m_pytest.log 2>&1; tail -3 gpurun_out/r2m_pytest.log
