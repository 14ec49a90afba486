timeout 300 python tools/profile_e.py 2 > gpurun_out/r2j_e.json 2>&1; cat gpurun_out/r2j_e.json | tail -2
# stage kernels of iteration 0/1: first, intensity, tail (2 iters) -> capture a tail launch and an intensity launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 1 -c 3 -o gpurun_out/r2j_e_stage python tools/profile_e.py 2 > gpurun_out/r2j_ncu.log 2>&1; tail -3 gpurun_out/r2j_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:apss_kernel -s 0 -c 1 -o gpurun_out/r2j_e_apss python tools/profile_e.py 1 > gpurun_out/r2j_ncu2.log 2>&1; tail -3 gpurun_out/r2j_ncu2.log
