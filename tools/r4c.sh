timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_dropin.py > gpurun_out/r4c_tests.log 2>&1; tail -2 gpurun_out/r4c_tests.log
BATCHES=1,16 KT=1 timeout 600 python tools/batch_probe.py B C 2>&1 | tail -8
timeout 300 python tools/profile_e.py 2 2>&1 | tail -1
