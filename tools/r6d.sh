for v in knn7 knn6 knn5; do RT3D_LIB=$PWD/ab/librt3d_$v.so BATCHES=1,16 KT=1 timeout 600 python tools/batch_probe.py B C 2>&1 | grep "kernel_ms\|ms_per_batch" | sed "s/^/$v /" | cut -c1-200; done
