for lib in paper_1905_06700_b200/librt3d.so ab_ilp.so; do
  echo "== $lib"
  RT3D_LIB=$PWD/$lib timeout 300 python tools/batch_probe.py B 2>&1 | grep -E '"batch": (1|8)'
  RT3D_LIB=$PWD/$lib timeout 300 python tools/profile_e.py 2 2>&1 | tail -1
done
