R=$GRAFT_REPO_ROOT; cd $R; O=$R/gpurun_out; mkdir -p $O
timeout 400 python -m pytest tests/test_replay_gpu.py -x -q > $O/ep_tests_e1.log 2>&1; echo "e1 tests rc=$?" >> $O/ep_tests_e1.log
rm -rf /tmp/r2; mkdir /tmp/r2; cp -r paper_2302_06173_b200 include tests oracle bench.py __graft_entry__.py /tmp/r2/; mkdir -p /tmp/r2/build/obj
(cd /tmp/r2/paper_2302_06173_b200/csrc && make -s -j32 EXTRA_NVFLAGS="-DRWB_GEMM2_CQ=2" > /dev/null 2>&1)
(cd /tmp/r2 && timeout 400 python -m pytest tests/test_replay_gpu.py -x -q > $O/ep_tests_cq2.log 2>&1; echo "cq2 tests rc=$?" >> $O/ep_tests_cq2.log)
for v in e0 e1 cq2; do timeout 120 tools/gpi_$v 1.0 wide > $O/ep_gpi_$v.log 2>&1; done
for r in 1 2; do for v in e0 e1 cq2; do echo "== $v" >> $O/ep_gp.log; timeout 120 tools/gp_$v 2.0 wide >> $O/ep_gp.log 2>&1; done; done
VARIANTS="e0:-DRWB_EPI_EARLY_RELEASE=0 e1: cq2:-DRWB_GEMM2_CQ=2" ROUNDS=2 timeout 1200 bash tools/gemm_variants.sh > $O/ep_variants.log 2>&1
