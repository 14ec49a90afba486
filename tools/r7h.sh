BATCHES=8,12,16,20,24 timeout 600 python tools/batch_probe.py B 2>&1 | tail -5
