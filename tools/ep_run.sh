#!/bin/bash
# epilogue A/B on one box: instrumented + timing GEMM probes of the wide pair
# kernel for each prebuilt variant (tools/gpi_<v>, tools/gp_<v>), then the
# config-4 replay under gemm_variants.sh.  usage: V="a b" VARIANTS="a:flags b:flags" bash tools/ep_run.sh tag
R=$GRAFT_REPO_ROOT; cd $R; O=$R/gpurun_out; mkdir -p $O; T=${1:-ep}
for v in $V; do echo "== $v" >> $O/${T}_gpi.log; timeout 120 tools/gpi_$v 1.0 wide >> $O/${T}_gpi.log 2>&1; done
for r in 1 2; do for v in $V; do echo "== $v" >> $O/${T}_gp.log; timeout 120 tools/gp_$v 2.0 wide >> $O/${T}_gp.log 2>&1; done; done
ROUNDS=2 timeout 1200 bash tools/gemm_variants.sh > $O/${T}_variants.log 2>&1
