timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_parity_configs.py tests/test_per_pixel_irf.py -q -x > gpurun_out/r3c_tests.log 2>&1; tail -2 gpurun_out/r3c_tests.log
for k in B C; do echo "== $k"; RT3D_LIB=$PWD/ab_prof.so timeout 300 python tools/sweep_profile.py $k 2>&1 | head -10; done
BATCHES=1,8,16 timeout 600 python tools/batch_probe.py B C 2>&1 | tail -6
