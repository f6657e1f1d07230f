"""Config 5: selective-logging sweep on a Llama-7B-shaped pipeline.

p = 8 stages, each = 4 Llama MLP blocks (4096 -> 11008 -> 4096) = 8 affine+tanh
layers (32 layers / 8 stages), micro-batch 8 x 2048 tokens = 16384 rows, m
micro-batches, Adam.  Selective logging with uniform groups of k stages
(PAPER:391 balanced grouping; "log every k-th stage boundary"): a failure
replays the k stages of its group from the logs at the group's boundaries.

For k in {1, 2, 4, 8} this measures, on this box's GPU(s):
  * log bytes per iteration  = (p/k - 1) boundaries x m x (activation + gradient)
  * replay ms per lost iteration of one failed group (tcgen05 GEMMs, logs in HBM)
and evaluates the SPEC planner (group_machines / recovery_time_estimate,
SPEC:567-584) on the measured per-stage replay time.

usage: python tools/c5_sweep.py [m] [out.json]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2302_06173_b200 import ADAM, OptimizerHyper, planner  # noqa: E402
from paper_2302_06173_b200.replay import BoundaryLog, Stage, replay_group, synth_inputs  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
out_path = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/c5_sweep.json"
p, R, H, F, blocks = 8, 16384, 4096, 11008, 4
dims = [H, F] * blocks + [H]
L = len(dims) - 1
h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
flop_stage_mb = sum(2 * R * dims[i] * dims[i + 1] for i in range(L)) * 3  # fwd + dgrad + wgrad
boundary_bytes = R * H * 2  # one bf16 boundary message (activation or gradient)
res = {"p": p, "rows": R, "micro_batches": m, "stage_dims": dims, "sweep": []}

for k in (1, 2, 4, 8):
    torch.cuda.empty_cache()
    stages = [Stage(s, H, F, H, L, 7, ADAM, dims=dims) for s in range(k)]  # group [0, k)
    last = k == p
    log = BoundaryLog()
    if not last:
        for mb in range(m):
            g = synth_inputs(9, 0, mb, R, H).mul_(1e-3)
            for it in range(2):
                log.grads[(it, mb)] = g
    replay_group(stages, log, 0, 1, R, m, 7, h, first=True, last=last, dim=H)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    replay_group(stages, log, 1, 2, R, m, 7, h, first=True, last=last, dim=H)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    flop = flop_stage_mb * m * k
    logged_boundaries = p // k - 1
    res["sweep"].append(dict(
        k=k, groups=p // k, logged_boundaries=logged_boundaries,
        log_bytes_per_iteration=logged_boundaries * m * 2 * boundary_bytes,
        replay_ms_per_lost_iteration=round(ms, 2), replay_tflops=round(flop / (ms * 1e-3) / 1e12, 1),
        wall_ms=round((time.perf_counter() - t0) * 1e3, 2)))
    print(json.dumps(res["sweep"][-1]), flush=True)
    del stages, log

# planner on the measured profile: R_i = per-stage replay seconds per lost iteration,
# M_i = bytes per iteration across boundary i, B = log-fetch bandwidth, T = checkpoint interval
r1 = res["sweep"][0]["replay_ms_per_lost_iteration"] / 1e3
M = [m * 2 * boundary_bytes] * (p - 1)
B, T = 25e9, 100
plans = []
for frac in (1.0, 0.5, 0.25, 0.0):
    Mmax = frac * T * sum(M)
    for par in (False, True):
        gp = planner.group_machines([r1] * p, M, B, T, Mmax, parallel=par)
        plans.append(dict(M_max_fraction=frac, parallel=par, groups=gp.groups, storage_bytes=gp.storage,
                          est_recovery_s_per_lost_iteration=round(gp.recovery, 4),
                          est_recovery_s_50_lost=round(
                              planner.recovery_time_estimate([r1] * p, M, B, gp.groups, 50, par), 3)))
res["planner"] = dict(R_stage_s=r1, boundary_bytes_per_iteration=M[0], B=B, T=T, plans=plans)
Path(out_path).parent.mkdir(exist_ok=True)
Path(out_path).write_text(json.dumps(res, indent=1))
print(json.dumps(res["planner"], indent=1))
