timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r7b_tests.log 2>&1; tail -3 gpurun_out/r7b_tests.log
timeout 600 python tools/e2e_probe.py 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r7b_bench.json 2> gpurun_out/r7b_bench.err; python -c "import json;d=json.load(open('gpurun_out/r7b_bench.json'));print(d['value'],d['e2e']['value'],d['details']['single_frame_fps'])"
