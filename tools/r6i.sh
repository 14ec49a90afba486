timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r6i_tests.log 2>&1; tail -1 gpurun_out/r6i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r6i_smoke.log 2>&1; tail -1 gpurun_out/r6i_smoke.log
timeout 1200 python bench.py > gpurun_out/r6i_bench.json 2> gpurun_out/r6i_bench.err; python -c "import json; d=json.loads(open('gpurun_out/r6i_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['details']['single_frame_fps'], d['roofline']['frac'], d['large_array']['ms_per_frame'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r6i_ref.json 2> gpurun_out/r6i_ref.err; tail -c 300 gpurun_out/r6i_ref.json
