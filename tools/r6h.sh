timeout 900 python -m pytest tests/test_batch.py tests/test_stream.py -m gpu -q > gpurun_out/r6h_tests.log 2>&1; tail -2 gpurun_out/r6h_tests.log
