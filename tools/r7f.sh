BATCHES=1,16 KT=1 timeout 600 python tools/batch_probe.py B C 2>&1 | tail -8
timeout 300 python tools/profile_e.py 2 2>&1 | tail -1
