"""B200-native RT3D reconstruction path (arXiv 1905.06700), drop-in for
splidar::reconstruct.  The compute lives in librt3d.so (CUDA, sm_100a) behind
the C ABI in include/rt3d.h; this package only loads it and binds it."""
