#!/bin/bash
# A/B the fused step/undo kernel's tiling on the GPU box: builds package copies
# with different (stages, slot bytes, min CTAs per SM) and times the Adam and
# AdamW undo at 336M and 1B in each.  usage: bash tools/optim_variants.sh
set -e
cd "$(dirname "$0")/.."
ROOT=$(pwd)
for v in ${VARIANTS:-"base:3:8192:1" "s4k4:4:4096:3" "s3k4:3:4096:3" "s6k4:6:4096:2"}; do
  IFS=: read name st sb mb <<< "$v"
  D=/tmp/optv/$name
  rm -rf $D; mkdir -p $D
  cp -r paper_2302_06173_b200 include $D/
  mkdir -p $D/build/obj
  (cd $D/paper_2302_06173_b200/csrc && make -s -j16 EXTRA_NVFLAGS="-DRW_OPTIM_STAGES=$st -DRW_OPTIM_SLOT_BYTES=$sb -DRW_OPTIM_MIN_BLOCKS=$mb" >/dev/null 2>&1) &
done
wait
for round in 1 2; do
for v in ${NAMES:-base s4k4 s3k4 s6k4}; do
  (cd /tmp && PYTHONPATH=/tmp/optv/$v:$ROOT python -) <<PY
import sys, statistics, json
import paper_2302_06173_b200 as P
assert P.__file__.startswith("/tmp/optv/$v"), P.__file__
import bench, torch
from paper_2302_06173_b200.workloads import CONFIGS
out = {}
for cfg, kind in (("adam340m", "adam"), ("adam340m", "adamw"), ("adam1b", "adam")):
    t, nb, st, _ = bench.measure_undo(CONFIGS[cfg]["sizes"](), kind, 8, 3)
    del st; torch.cuda.empty_cache()
    out[f"{cfg}-{kind}"] = round(statistics.median(t), 4)
print("$v", json.dumps(out), flush=True)
PY
done
done
