timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_parity_configs.py tests/test_spatial_grid.py tests/test_batch.py -m gpu -q -x > gpurun_out/r3j_tests.log 2>&1; tail -2 gpurun_out/r3j_tests.log
BATCHES=1,16 KT=1 timeout 600 python tools/batch_probe.py B C 2>&1 | tail -8
timeout 300 python tools/profile_e.py 2 2>&1 | tail -1
