timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r5o_tests.log 2>&1; tail -1 gpurun_out/r5o_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5o_smoke.log 2>&1; tail -2 gpurun_out/r5o_smoke.log
timeout 1200 python bench.py > gpurun_out/r5o_bench.json 2> gpurun_out/r5o_bench.err; tail -c 300 gpurun_out/r5o_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r5o_ref.json 2> gpurun_out/r5o_ref.err; tail -c 400 gpurun_out/r5o_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r5o_launches.csv python tools/profile_batch.py B 16 > gpurun_out/r5o_l.log 2>&1; tail -1 gpurun_out/r5o_l.log
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -c 8 -f -o gpurun_out/r5o_full python tools/profile_batch.py B 16 > gpurun_out/r5o_f.log 2>&1; tail -1 gpurun_out/r5o_f.log
