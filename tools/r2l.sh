timeout 1200 oracle/_ref/ref_tests > gpurun_out/r2l_reftests.log 2>&1; echo "rc=$?"; grep -E "FAILED|test cases" -A2 gpurun_out/r2l_reftests.log | head -60
for c in 1 2 3 4 5 6 7 8; do timeout 600 oracle/_ref/ref_acceptance $c > gpurun_out/r2l_acc$c.log 2>&1; echo "C$c rc=$?"; tail -3 gpurun_out/r2l_acc$c.log; done
