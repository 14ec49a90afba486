timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r5s_tests.log 2>&1; tail -3 gpurun_out/r5s_tests.log
