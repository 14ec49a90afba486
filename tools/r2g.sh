timeout 900 python -m pytest tests/test_batch.py -q -x > gpurun_out/r2g_batch.log 2>&1; tail -15 gpurun_out/r2g_batch.log
timeout 900 python tools/batch_probe.py B C > gpurun_out/r2g_probe.jsonl 2> gpurun_out/r2g_probe.err; cat gpurun_out/r2g_probe.jsonl; tail -3 gpurun_out/r2g_probe.err
