timeout 900 python -m pytest tests/test_stream.py tests/test_per_pixel_irf.py -q -x -rA > gpurun_out/r2b_new.log 2>&1; tail -12 gpurun_out/r2b_new.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_parity_configs.py > gpurun_out/r2b_pytest.log 2>&1; tail -4 gpurun_out/r2b_pytest.log
timeout 900 python bench.py --no-parity > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; tail -3 gpurun_out/r2b_bench.err; python -c "
import json;d=json.load(open('gpurun_out/r2b_bench.json'));print(d['value'],d['e2e']['value'])"
