timeout 1200 python bench.py > gpurun_out/r7i_bench.json 2> gpurun_out/r7i_bench.err; tail -c 200 gpurun_out/r7i_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r7i_launches.csv python tools/profile_batch.py B 20 > gpurun_out/r7i_l.log 2>&1; tail -1 gpurun_out/r7i_l.log
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -c 8 -f -o gpurun_out/r7i_full python tools/profile_batch.py B 20 > gpurun_out/r7i_f.log 2>&1; tail -1 gpurun_out/r7i_f.log
