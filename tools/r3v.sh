BATCHES=1,16 KT=1 timeout 600 python tools/batch_probe.py C 2>&1 | tail -4
