timeout 600 python tools/group_probe.py B 2>&1 | tail -4
timeout 600 python tools/group_probe.py C 2>&1 | tail -4
RT3D_TWO_CAND=3 timeout 300 python tools/batch_probe.py C 2>&1 | tail -4
