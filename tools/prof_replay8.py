"""Kernel-time breakdown of one replayed iteration of the config-4 8-stage
group on one GPU, with torch.profiler (CUPTI activity records: real
concurrent timings, unlike ncu's serialised replay)."""
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.append(str(Path(__file__).resolve().parents[1]))  # a PYTHONPATH build variant wins

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2302_06173_b200 import ADAM, OptimizerHyper  # noqa: E402
from paper_2302_06173_b200.replay import BoundaryLog, Stage, replay_group, synth_inputs  # noqa: E402

n_stages = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rows, m, dims = 16384, 8, (4096, 16384, 4096)
h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
sts = [Stage(s, dims[0], dims[1], dims[2], 2, 2302, ADAM) for s in range(n_stages)]
log = BoundaryLog()
for mb in range(m):
    a = synth_inputs(5, 0, mb, rows, dims[0])
    g = synth_inputs(6, 0, mb, rows, dims[-1]).mul_(1e-3)
    for it in range(3):
        log.acts[(it, mb)] = a
        log.grads[(it, mb)] = g
replay_group(sts, log, 0, 1, rows, m, 2302, h, first=False, last=False, dim=dims[0])
torch.cuda.synchronize()
t0 = time.perf_counter()
replay_group(sts, log, 1, 2, rows, m, 2302, h, first=False, last=False, dim=dims[0])
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    replay_group(sts, log, 2, 3, rows, m, 2302, h, first=False, last=False, dim=dims[0])
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
first, last = None, None
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    k = e.name[:90]
    agg[k][0] += 1
    agg[k][1] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else e.cuda_time_total / 1e3
    s, t = e.time_range.start, e.time_range.end
    first = s if first is None else min(first, s)
    last = t if last is None else max(last, t)
busy = sum(v for _, v in agg.values())
print(f"stages={n_stages} wall(no profiler)={wall:.1f} ms  gpu span={(last - first) / 1e3:.1f} ms  kernel sum={busy:.1f} ms")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{v:9.2f} ms {v / busy * 100:5.1f}% x{n:4d} {k}")
