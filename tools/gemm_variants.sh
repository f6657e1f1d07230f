#!/bin/bash
# A/B of the replay GEMM's build options under sustained (power-capped) load:
# builds package copies with different EXTRA_NVFLAGS (raster group, barrier
# suspend hint, ...) and, alternating, times the config-4 replay (one
# iteration of the 8-stage group, bench.replay_bench) and the forward stage
# against cuBLAS (tools/sustained_gemm.py).
# usage: VARIANTS="name:flag1+flag2 ..." ROUNDS=2 bash tools/gemm_variants.sh
set -e
cd "$(dirname "$0")/.."
ROOT=$(pwd)
VARIANTS=${VARIANTS:-"base:"}
NAMES=""
for v in $VARIANTS; do
  IFS=: read name xf <<< "$v"; XF=$(echo "$xf" | tr "+" " ")
  NAMES="$NAMES $name"
  D=/tmp/gemmv/$name
  rm -rf $D; mkdir -p $D
  cp -r paper_2302_06173_b200 include $D/
  mkdir -p $D/build/obj
  (cd $D/paper_2302_06173_b200/csrc && make -s -j16 EXTRA_NVFLAGS="$XF" >/dev/null 2>&1) &
done
wait
for round in $(seq 1 ${ROUNDS:-2}); do
for v in $NAMES; do
  (cd /tmp && PYTHONPATH=/tmp/gemmv/$v:$ROOT python -) <<PY
import json, torch
import paper_2302_06173_b200 as P
assert P.__file__.startswith("/tmp/gemmv/$v"), P.__file__
import bench
r = bench.replay_bench(1, 0, torch.device("cuda", 0), iters=2)
print("$v", json.dumps(dict(replay_ms=r["ms_per_iteration"], tflops=r["tflops_aggregate"])), flush=True)
PY
  (cd /tmp && PYTHONPATH=/tmp/gemmv/$v:$ROOT python $ROOT/tools/sustained_gemm.py 3 | python -c "
import json,sys; d=json.load(sys.stdin); print('$v sustained', {k: (v['tflops'], v['clocks'].get('sm_mhz')) for k, v in d.items()})")
done
done
