timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r7e_ref.json 2> gpurun_out/r7e_ref.err; tail -c 600 gpurun_out/r7e_ref.json
