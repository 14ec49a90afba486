BATCHES=1,16 timeout 300 python tools/batch_probe.py B C 2>&1 | tail -4 | sed "s/^/default /"
RT3D_TWO_CAND=3 BATCHES=1,16 timeout 300 python tools/batch_probe.py B C 2>&1 | tail -4 | sed "s/^/two3 /"
