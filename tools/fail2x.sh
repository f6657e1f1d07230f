cd $GRAFT_REPO_ROOT
for i in 1 2 3 4 5 6; do echo "== run $i" >> gpurun_out/fail2x.log; timeout -s KILL 200 tests/cpp/recover_host_test failure 2 >> gpurun_out/fail2x.log 2>&1; echo "rc=$?" >> gpurun_out/fail2x.log; done
timeout 1200 python -m pytest tests/test_recover_host_gpu.py -x -q > gpurun_out/recover_host_tests_n2.log 2>&1
