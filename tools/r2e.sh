timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2e_pytest.log 2>&1; tail -3 gpurun_out/r2e_pytest.log
CHECK_ITERS=0 timeout 900 python tools/bench_configs.py 3 D E > gpurun_out/r2e_de.jsonl 2> gpurun_out/r2e_de.err; cat gpurun_out/r2e_de.jsonl
timeout 900 python bench.py --no-parity --no-cpu-baseline > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; tail -2 gpurun_out/r2e_bench.err; python -c "
import json;d=json.load(open('gpurun_out/r2e_bench.json'));print(d['value'],d['e2e']['value']);print({k:(round(v['ms_per_frame'],3), v['us_per_launch']) for k,v in d['kernel_classes'].items() if v['us_per_launch']})"
