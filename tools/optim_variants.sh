#!/bin/bash
# A/B the fused step/undo kernel's build options on the GPU box: builds package
# copies with different (stages, slot bytes, min CTAs per SM, interleaved tile
# order, L2 eviction hint) and times the Adam undo/step at 336M and 1B in each,
# next to a torch copy of the same box (the measured-peak recipe).
# usage: VARIANTS="name:st:slot:minb:il:l2 ..." bash tools/optim_variants.sh
set -e
cd "$(dirname "$0")/.."
ROOT=$(pwd)
VARIANTS=${VARIANTS:-"base:3:8192:1:0:0 il:3:8192:1:1:0 l2:3:8192:1:0:2 il_l2:3:8192:1:1:2"}
NAMES=""
for v in $VARIANTS; do
  IFS=: read name st sb mb il l2 xf <<< "$v"; XF=$(echo "$xf" | tr "+" " ")
  NAMES="$NAMES $name"
  D=/tmp/optv/$name
  rm -rf $D; mkdir -p $D
  cp -r paper_2302_06173_b200 include $D/
  mkdir -p $D/build/obj
  (cd $D/paper_2302_06173_b200/csrc && make -s -j16 EXTRA_NVFLAGS="-DRW_OPTIM_STAGES=$st -DRW_OPTIM_SLOT_BYTES=$sb -DRW_OPTIM_MIN_BLOCKS=$mb -DRW_OPTIM_INTERLEAVE=$il -DRW_OPTIM_L2HINT=$l2 $XF" >/dev/null 2>&1) &
done
wait
python - <<'PY'
import torch
a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda"); b = torch.empty_like(a)
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); b.copy_(a); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
print("copy_peak_gbs", round(4 * (1 << 30) / best / 1e6, 1), flush=True)
PY
for round in $(seq 1 ${ROUNDS:-3}); do
for v in $NAMES; do
  (cd /tmp && PYTHONPATH=/tmp/optv/$v:$ROOT python -) <<PY
import sys, statistics, json
import paper_2302_06173_b200 as P
assert P.__file__.startswith("/tmp/optv/$v"), P.__file__
import bench, torch
from paper_2302_06173_b200.workloads import CONFIGS
out = {}
for cfg, kind in (("adam340m", "adam"), ("adam1b", "adam")):
    t, nb, st, _ = bench.measure_undo(CONFIGS[cfg]["sizes"](), kind, 8, 3)
    del st; torch.cuda.empty_cache()
    out[f"{cfg}-undo"] = round(nb / statistics.median(t) / 1e6, 1)
    out[f"{cfg}-step"] = round(nb / statistics.median(bench.measure_undo.last_step_ms) / 1e6, 1)
print("$v", json.dumps(out), flush=True)
PY
done
done
