#!/bin/bash
# GPU tests + a short bench, printing the per-kernel-class breakdown
python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; tail -4 gpurun_out/pytest.log
python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read())
print("value", round(d["value"], 2), "e2e", round(d["e2e"]["value"], 2), "ms", round(d["ms_per_step"], 3))
for c, v in d["kernel_classes"].items():
    if v["us_per_launch"] is None:
        continue
    print(f'{c:16s} {v["ms_per_frame"]:.3f} ms/frame  {v["us_per_launch"]:.1f} us/launch')
PY
