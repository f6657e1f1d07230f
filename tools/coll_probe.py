"""Latency of the small host-side steps of a recovery call (torchrun, NCCL):
all_gather_object of IPC handles, barrier, marker broadcast + D2H."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch
import torch.distributed as dist

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
from paper_2302_06173_b200.recovery import _export  # noqa: E402

bufs = [torch.empty(1 << 20, device=dev) for _ in range(4)]
res = {}


def t(name, fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    res[name] = round((time.perf_counter() - t0) / n * 1e3, 3)


def ago():
    out = [None] * world
    dist.all_gather_object(out, dict(bufs={i: _export(b) for i, b in enumerate(bufs)}))


t("all_gather_object_handles_ms", ago)
t("barrier_ms", lambda: dist.barrier())
mk = torch.zeros(1160, dtype=torch.int64, device=dev)
t("marker_broadcast_plus_d2h_ms", lambda: (dist.broadcast(mk, src=0), mk.cpu().tolist()))
t("export_4_handles_ms", lambda: [_export(b) for b in bufs])
if rank == 0:
    print(json.dumps(res))
dist.destroy_process_group()
