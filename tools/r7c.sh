timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r7c_tests.log 2>&1; tail -3 gpurun_out/r7c_tests.log
timeout 900 python bench.py > gpurun_out/r7c_bench.json 2> gpurun_out/r7c_bench.err; python -c "import json;d=json.load(open('gpurun_out/r7c_bench.json'));print(d['value'],d['e2e']['value'],d['details']['single_frame_fps'])"
timeout 900 python bench.py --no-parity --no-large --no-cpu-baseline --e2e-groups 1 > gpurun_out/r7c_1.json 2> gpurun_out/r7c_1.err; python -c "import json;d=json.load(open('gpurun_out/r7c_1.json'));print('groups1', d['value'],d['e2e']['value'])"
