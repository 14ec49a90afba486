RT3D_KNN_W0=9 BATCHES=16 KT=1 timeout 600 python tools/batch_probe.py B 2>&1 | grep "kernel_ms" | cut -c1-220
