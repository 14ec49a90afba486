BATCHES=1,8,12,16 timeout 600 python tools/batch_probe.py B C 2>&1 | tail -8
