nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_gpu.txt
timeout 1500 python -m pytest tests/test_parity_configs.py -q -x -rA > gpurun_out/r2a_parity.log 2>&1; tail -30 gpurun_out/r2a_parity.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_parity_configs.py > gpurun_out/r2a_pytest.log 2>&1; tail -4 gpurun_out/r2a_pytest.log
timeout 900 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -3 gpurun_out/r2a_bench.err; head -c 600 gpurun_out/r2a_bench.json
