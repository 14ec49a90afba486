timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "fft" > gpurun_out/r2v_fft.log 2>&1; tail -3 gpurun_out/r2v_fft.log
timeout 600 python tools/fft_probe.py 2>&1 | tail -5
