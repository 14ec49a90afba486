timeout 900 python bench.py --no-parity --no-cpu-baseline --no-large > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err; tail -2 gpurun_out/r2x_bench.err; python -c "
import json;d=json.load(open('gpurun_out/r2x_bench.json'));print(d['value'],d['e2e'])"
RT3D_GSZ=1 timeout 300 python tools/batch_probe.py B 2>&1 | grep -E '"batch": (1|8)'
