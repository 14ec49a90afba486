for lib in paper_1905_06700_b200/librt3d.so ab_g1b4.so; do
  RT3D_LIB=$PWD/$lib timeout 300 python tools/profile_e.py 3 2>&1 | tail -1
done
