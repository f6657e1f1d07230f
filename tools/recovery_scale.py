"""Config-3 replica recovery alone at N GPUs (torchrun): bench.recovery_e2e."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2302_06173_b200 import recovery as _rec  # noqa: E402

if os.environ.get("RW_CHAIN"):  # sweep hook: "pieces,split" of the copy-engine chain
    _p, _s = (int(v) for v in os.environ["RW_CHAIN"].split(","))
    _d = list(_rec.recover_replication_chain.__defaults__)
    _d[-2], _d[-1] = _p, _s
    _rec.recover_replication_chain.__defaults__ = tuple(_d)
if os.environ.get("RW_MODES"):
    bench.RECOVERY_MODES = os.environ["RW_MODES"].split(",")

rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(
    os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
r = bench.recovery_e2e(world, rank, dev)
if rank == 0:
    print(json.dumps({k: (v.get("recovery_ms"), v.get("resolve_ms"), v.get("transfer")) if isinstance(v, dict) else v
                      for k, v in r.items()}), flush=True)
if world > 1:
    dist.destroy_process_group()
