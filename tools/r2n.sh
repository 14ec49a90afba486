timeout 900 python -m pytest tests/test_spatial_grid.py -q -x > gpurun_out/r2n_grid.log 2>&1; tail -5 gpurun_out/r2n_grid.log
for lib in paper_1905_06700_b200/librt3d.so ab_apss5.so ab_apss6.so; do
  echo "== $lib"
  RT3D_LIB=$PWD/$lib timeout 300 python tools/batch_probe.py B 2>&1 | grep '"batch": 8'
  RT3D_LIB=$PWD/$lib timeout 300 python tools/profile_e.py 2 2>&1 | tail -1
done
