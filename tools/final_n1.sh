#!/bin/bash
# Round-end evidence on one GPU: the GPU suite, smoke(), the default bench line.
T=${1:-final}; cd $GRAFT_REPO_ROOT; O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest_n1_${T}.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_${T}.log 2>&1
timeout 1200 python bench.py > $O/bench_n1_${T}.json 2> $O/bench_n1_${T}.err
cp $O/bench_extras.json $O/bench_n1_${T}_extras.json 2>/dev/null
timeout 900 python bench.py --impl reference > $O/bench_ref_${T}.json 2> $O/bench_ref_${T}.err
