#!/bin/bash
# One GPU call's worth of round-end evidence (run on the box, one GPU):
#   bench line, the bench's kernel launch list, ncu --set full of one 1B Adam
#   undo launch and of the four replay GEMMs of one micro-batch.
# usage: bash tools/profile_round.sh <tag>     (writes gpurun_out/<tag>_*)
set -x
T=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline \
  > $O/${T}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim_kernel -s 3 -c 1 \
  -o $O/${T}_undo1b -f python tools/prof_undo.py adam1b > $O/${T}_undo1b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_gemm -s 32 -c 4 \
  -o $O/${T}_replay_gemms -f python tools/prof_replay.py 1 > $O/${T}_replay_gemms.log 2>&1
ls -la $O
