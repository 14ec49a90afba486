timeout 600 python tools/e2e_probe.py 2>&1 | tail -2
timeout 900 ncu --nvtx --nvtx-include "rt3d_state_copy/" --metrics gpu__time_duration.sum --clock-control none -c 3 --csv --log-file gpurun_out/r7a_nvtx.csv python tools/e2e_probe.py > gpurun_out/r7a_nvtx.log 2>&1; tail -2 gpurun_out/r7a_nvtx.log; grep -c gather gpurun_out/r7a_nvtx.csv; grep -v gather gpurun_out/r7a_nvtx.csv | grep -c duration
