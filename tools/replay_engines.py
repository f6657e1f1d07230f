"""A/B of the replay GEMM engine on the config-4 replay (bench.replay_bench,
N=1): single-CTA tcgen05 kernel vs the CTA-pair (cta_group::2, M=256)
kernel, both with the TMA epilogue, alternating, so both see the same
power-capped board.  usage: python tools/replay_engines.py [rounds]"""
import sys
from pathlib import Path

sys.path.append(str(Path(__file__).resolve().parents[1]))  # a PYTHONPATH build variant wins
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2302_06173_b200.replay import LIB  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda", 0)
for r in range(rounds):
    for pair in (0, 1, 2):
        assert LIB.rw_replay_set_gemm_engine(1, pair) == 0
        out = bench.replay_bench(1, 0, dev, iters=2)
        print(f"round {r} pair={pair} ms/iter {out['ms_per_iteration']} TFLOP/s {out['tflops_aggregate']}",
              flush=True)
