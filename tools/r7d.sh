timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r7d_tests.log 2>&1; tail -25 gpurun_out/r7d_tests.log | grep -v "^\.\.\." | tail -15
BATCHES=1,16 KT=1 timeout 600 python tools/batch_probe.py B C 2>&1 | tail -8
timeout 300 python tools/profile_e.py 2 2>&1 | tail -1
