timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4e_tests.log 2>&1; tail -2 gpurun_out/r4e_tests.log
timeout 900 python bench.py > gpurun_out/r4e_bench.json 2> gpurun_out/r4e_bench.err; tail -c 3000 gpurun_out/r4e_bench.json
