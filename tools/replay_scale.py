"""Config-4 replay alone at N GPUs (torchrun), for scaling experiments:
prints bench.replay_bench's dict on rank 0."""
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
it = int(sys.argv[1]) if len(sys.argv) > 1 else 2
r = bench.replay_bench(world, rank, dev, iters=it)
torch.cuda.empty_cache()
r2 = bench.replay_subpipeline_bench(world, rank, dev, iters=it) if world > 1 else None
if rank == 0:
    print(json.dumps(dict(parallel=r["ms_per_iteration"], subpipeline=r2 and r2["ms_per_iteration"],
                          bubble=r2 and r2["pipeline_bubble"])), flush=True)
if world > 1:
    dist.destroy_process_group()
