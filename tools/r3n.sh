timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_dropin.py > gpurun_out/r3n_tests.log 2>&1; tail -2 gpurun_out/r3n_tests.log
BATCHES=1,16 KT=1 timeout 600 python tools/batch_probe.py C 2>&1 | tail -4
