timeout 1200 python bench.py > gpurun_out/r7j_bench.json 2> gpurun_out/r7j_bench.err; tail -c 300 gpurun_out/r7j_bench.json
