"""Copy-engine chain transfer (recovery.recover_replication_chain, N=2) of the
GPT-2 XL state timed transfer by transfer: warm-up transfers without undo,
then transfers right after the survivor's SMs rewrote the state (a step over
half the groups), to see whether a transfer after kernel writes runs slower.
torchrun --nproc-per-node 2 tools/chain_cold_probe.py"""
import os
import sys
import time

sys.path.append(os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper  # noqa: E402
from paper_2302_06173_b200.recovery import recover_replication_chain, resolve  # noqa: E402
from paper_2302_06173_b200.workloads import gpt2_xl_sizes  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
sizes = gpt2_xl_sizes()
st = DeviceState(sizes, kind=ADAM, device=rank)
h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
if rank == 0:
    for t in (st.x, st.g, st.m, st.v):
        t.uniform_(-0.1, 0.1)
    st.v.abs_()
    st.write_markers([(10, 0)] * st.num_groups)


def transfer(tag):
    torch.cuda.synchronize()
    dist.barrier()
    plan = resolve(st.markers() if rank == 0 else [], h, lens=sizes if rank == 0 else None, device=dev)
    t0 = time.perf_counter()
    recover_replication_chain(st, h, plan, src=0)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    if rank == 0:
        print(f"{tag}: strategy {plan.strategy} {ms:.2f} ms", flush=True)


for i in range(3):
    transfer(f"warm {i}")
for i in range(3):
    if rank == 0:  # SM writes: one step of half the groups, then the markers re-armed as healthy
        st.step(h, stop_after=st.num_groups // 2)
        st.write_markers([(10, 0)] * st.num_groups)
    transfer(f"after step {i}")
for i in range(2):
    transfer(f"again {i}")
for i in range(3):
    if rank == 0:
        st.write_markers([(10, 0)] * st.num_groups)
        st.step(h, stop_after=st.num_groups // 2)
    transfer(f"undo+chain {i}")  # the survivor undoes inside the chain
dist.destroy_process_group()
