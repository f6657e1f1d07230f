"""NCCL broadcast of a GPT-2 XL-sized state (3 x 6.23 GB fp32) from rank 0
under different communicator configs (torchrun, N ranks)."""
import json
import os
import time

import torch
import torch.distributed as dist

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
n = 1_557_611_200
bufs = [torch.full((n,), float(rank), device=dev) for _ in range(3)]
res = {}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    best = 1e9
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    t = torch.tensor([best], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) * 1e3


res["default"] = timed(lambda: [dist.broadcast(b, 0) for b in bufs])
for cfg in ((16, 32), (32, 64), (64, 64)):
    o = dist.ProcessGroupNCCL.Options()
    o.config.min_ctas, o.config.max_ctas = cfg
    g = dist.new_group(backend="nccl", pg_options=o)
    res[f"ctas{cfg}"] = timed(lambda: [dist.broadcast(b, 0, group=g) for b in bufs])
# one broadcast per buffer, each on its own communicator -> concurrent
gs = [dist.new_group(backend="nccl") for _ in range(3)]
res["3comms_async"] = timed(lambda: [w.wait() for w in [dist.broadcast(b, 0, group=g, async_op=True)
                                                        for b, g in zip(bufs, gs)]])
if rank == 0:
    print(json.dumps({k: round(v, 2) for k, v in res.items()}), flush=True)
dist.destroy_process_group()
