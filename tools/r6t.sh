BATCHES=16 KT=1 timeout 600 python tools/batch_probe.py B 2>&1 | grep "kernel_ms\|ms_per_batch" | sed "s/^/default /" | cut -c1-220
RT3D_GSZ=3 BATCHES=16 KT=1 timeout 600 python tools/batch_probe.py B 2>&1 | grep "kernel_ms\|ms_per_batch" | sed "s/^/gsz3 /" | cut -c1-220
RT3D_GSZ=4 BATCHES=16 KT=1 timeout 600 python tools/batch_probe.py B 2>&1 | grep "kernel_ms\|ms_per_batch" | sed "s/^/gsz4 /" | cut -c1-220
