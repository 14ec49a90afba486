for w in 1 2 3; do RT3D_KNN_W0=$w BATCHES=16 KT=1 timeout 600 python tools/batch_probe.py B C 2>&1 | grep kernel_ms | sed "s/^/w0=$w /" | cut -c1-200; done
