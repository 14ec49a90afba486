timeout 900 python -m pytest tests/test_bands.py tests/test_batch.py -q -x > gpurun_out/r2i_bands.log 2>&1; tail -25 gpurun_out/r2i_bands.log
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_parity_configs.py > gpurun_out/r2i_pytest.log 2>&1; tail -3 gpurun_out/r2i_pytest.log
