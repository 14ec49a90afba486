BATCHES=1,16 timeout 600 python tools/batch_probe.py B 2>&1 | tail -2
