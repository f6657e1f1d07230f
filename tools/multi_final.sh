#!/bin/bash
# Multi-GPU evidence on one box of N GPUs: the >= 2-GPU tests, then the bench
# line at N (torchrun, one rank per GPU).  usage: bash tools/multi_final.sh <N> <tag>
N=${1:-2}; T=${2:-final}
cd $GRAFT_REPO_ROOT; O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_membership_gpu.py tests/test_recover_host_gpu.py -x -q \
  > $O/gputest_n${N}_${T}.log 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29631 bench.py --gpus $N > $O/bench_n${N}_${T}.json 2> $O/bench_n${N}_${T}.err
cp $O/bench_extras.json $O/bench_n${N}_${T}_extras.json 2>/dev/null
