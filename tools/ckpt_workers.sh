#!/bin/bash
# Checkpoint write / load rate by I/O worker count (RW_CKPT_WORKERS build option),
# alternating package copies on one box.  usage: bash tools/ckpt_workers.sh "8 16" [rounds]
cd "$(dirname "$0")/.."; ROOT=$(pwd)
for w in $1; do
  D=/tmp/ckptv/w$w; rm -rf $D; mkdir -p $D; cp -r paper_2302_06173_b200 include $D/; mkdir -p $D/build/obj
  (cd $D/paper_2302_06173_b200/csrc && make -s -j16 EXTRA_NVFLAGS="-DRW_CKPT_WORKERS=$w" >/dev/null 2>&1) &
done; wait
for r in $(seq 1 ${2:-2}); do for w in $1; do
  (cd /tmp && PYTHONPATH=/tmp/ckptv/w$w:$ROOT python -c "
import json, paper_2302_06173_b200 as P
assert P.__file__.startswith('/tmp/ckptv/w$w'), P.__file__
import bench
from paper_2302_06173_b200.workloads import CONFIGS
r = bench.checkpoint_bench(CONFIGS['adam340m']['sizes']())
print('workers $w', json.dumps({k: r[k] for k in ('write_gbs', 'load_gbs', 'bit_exact')}), flush=True)")
done; done
