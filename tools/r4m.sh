RT3D_SYNC_EACH=1 timeout 300 python tools/dbg_d.py D 2>&1 | tail -1 | cut -c1-100; RT3D_SYNC_EACH=1 timeout 300 python tools/dbg_d.py A 2>&1 | tail -1 | cut -c1-100
