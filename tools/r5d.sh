BATCHES=16,32 timeout 600 python tools/batch_probe.py B C 2>&1 | tail -4
