timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r7k_tests.log 2>&1; tail -1 gpurun_out/r7k_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
