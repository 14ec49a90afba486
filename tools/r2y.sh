timeout 900 python -m pytest tests/test_batch.py tests/test_bands.py tests/test_parity_configs.py -q -x > gpurun_out/r2y_tests.log 2>&1; tail -2 gpurun_out/r2y_tests.log
for env in "X=1" "RT3D_NBR_STRIDED=1"; do
  echo "== $env"
  env $env timeout 300 python tools/batch_probe.py B 2>&1 | grep -E '"batch": (1|8)'
  env $env timeout 300 python tools/profile_e.py 2 2>&1 | tail -1
done
