"""Config-3 replica recovery alone at N GPUs (torchrun): bench.recovery_e2e."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402

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
