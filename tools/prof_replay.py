"""Profiling driver: one replayed iteration of the config-4 stage on one GPU
(2 affine+tanh layers 4096->16384->4096, 8 micro-batches x 16384 rows, Adam)."""
import sys
import time
from pathlib import Path

sys.path.append(str(Path(__file__).resolve().parents[1]))  # a PYTHONPATH build variant wins

import torch  # noqa: E402

from paper_2302_06173_b200 import ADAM, OptimizerHyper  # noqa: E402
from paper_2302_06173_b200.replay import BoundaryLog, Stage, replay_group, synth_inputs  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rows, m, dims = 16384, 8, (4096, 16384, 4096)
h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
st = Stage(3, dims[0], dims[1], dims[2], 2, 2302, ADAM)
log = BoundaryLog()
for mb in range(m):
    a = synth_inputs(5, 0, mb, rows, dims[0])
    g = synth_inputs(6, 0, mb, rows, dims[-1]).mul_(1e-3)
    for it in range(iters + 1):
        log.acts[(it, mb)] = a
        log.grads[(it, mb)] = g
replay_group([st], log, 0, 1, rows, m, 2302, h, first=False, last=False, dim=dims[0])
torch.cuda.synchronize()
t0 = time.perf_counter()
replay_group([st], log, 1, 1 + iters, rows, m, 2302, h, first=False, last=False, dim=dims[0])
torch.cuda.synchronize()
print(f"prof_replay: {(time.perf_counter() - t0) * 1e3 / iters:.2f} ms/iteration")
