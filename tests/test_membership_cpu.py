"""Failure detection + communicator repair (membership.py) end to end on CPU
with gloo: three ranks, one crashes (os._exit), the survivors detect it from
its stopped heartbeat, abort the group, publish the repair plan, a fresh
replacement process claims the dead rank's slot, everyone joins generation
1, and the resolver + replica broadcast (the same code the B200 path runs
over NCCL) hand the replacement a bit-exact copy of the resolved state."""
import os
import socket
import time

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2302_06173_b200 import ADAM, OptimizerHyper
from paper_2302_06173_b200.membership import (Membership, abort_group, claim_slot, join_generation)
from paper_2302_06173_b200.recovery import recover_replication, resolve


class HostState:
    def __init__(self, sizes, seed=None):
        n = sum(sizes)
        g = torch.Generator().manual_seed(seed or 0)
        mk = (lambda: torch.randn(n, generator=g)) if seed is not None else (lambda: torch.zeros(n))
        self.device = torch.device("cpu")
        self.x, self.g, self.m, self.v = mk(), mk(), mk(), mk()
        self._mk = [(0, 0)] * len(sizes)

    def markers(self, stream=None):
        return list(self._mk)

    def write_markers(self, mk, stream=None):
        self._mk = [tuple(p) for p in mk]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SIZES = [5, 5, 5]


def _member(rank, port, q):
    store = dist.TCPStore("127.0.0.1", port, is_master=False, timeout=__import__("datetime").timedelta(seconds=60))
    from paper_2302_06173_b200.membership import RepairPlan
    join_generation(store, RepairPlan(0, 3, []), rank, "gloo")
    dist.barrier()
    mem = Membership(store, rank, 3, generation=0, interval=0.05, timeout=0.6)
    dist.barrier()  # every heartbeat is running
    h = OptimizerHyper(kind=ADAM)
    st = HostState(SIZES, seed=3)
    if rank == 2:  # fail-stop in the middle of the iteration
        store.set("crash_time", repr(time.time()))
        os._exit(1)
    # survivors: torn markers (rank 0 updated groups 2, 1; rank 1 only group 2)
    st.write_markers([(10, 0), (11, 1), (11, 1)] if rank == 0 else [(10, 0), (10, 0), (11, 1)])
    failed = mem.wait_failure(timeout=20)
    t_detect = mem.detected_at
    abort_group()
    plan = mem.publish_plan(settle=0.2)
    mem.stop()
    join_generation(store, plan, rank, "gloo")
    p = resolve(st.markers(), h, lens=SIZES)
    if rank == 0:
        st.write_markers([(10, 0)] * 3)  # apply_resolution (undo on the device path)
    nbytes = recover_replication(st, src=0)
    # numpy, not tensors: a torch queue shares tensors by fd and this process may exit first
    q.put((rank, dict(failed=sorted(failed), plan=plan.__dict__, strategy=p.strategy, target=p.target,
                      undo=p.undo_ids, x=st.x.numpy().copy(), mk=st.markers(), t_detect=t_detect,
                      crash=float(store.get("crash_time")), nbytes=nbytes)))
    dist.destroy_process_group()


def _replacement(port, q):
    store = dist.TCPStore("127.0.0.1", port, is_master=False, timeout=__import__("datetime").timedelta(seconds=60))
    plan, rank = claim_slot(store, 0)
    join_generation(store, plan, rank, "gloo")
    h = OptimizerHyper(kind=ADAM)
    p = resolve([], h)
    st = HostState(SIZES)
    recover_replication(st, src=0)
    q.put(("replacement", dict(rank=rank, x=st.x.numpy().copy(), mk=st.markers(), strategy=p.strategy)))
    dist.destroy_process_group()


def test_crash_detect_repair_and_recover():
    port = _free_port()
    store = dist.TCPStore("127.0.0.1", port, is_master=True, wait_for_workers=False)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_member, args=(r, port, q)) for r in range(3)]
    for p in ps:
        p.start()
    rep = ctx.Process(target=_replacement, args=(port, q))
    rep.start()
    res = dict(q.get(timeout=120) for _ in range(3))
    for p in ps + [rep]:
        p.join(timeout=60)
    assert ps[2].exitcode == 1  # the crashed rank
    assert ps[0].exitcode == 0 and ps[1].exitcode == 0 and rep.exitcode == 0
    a, b, r = res[0], res[1], res["replacement"]
    assert a["failed"] == b["failed"] == [2]
    assert a["plan"]["generation"] == 1 and a["plan"]["failed"] == [2] and a["plan"]["survivors"] == [0, 1]
    assert r["rank"] == 2
    assert a["strategy"] == b["strategy"] == r["strategy"] == "Undo" and a["target"] == 10
    assert a["undo"] == [1, 2] and b["undo"] == [2]
    for other in (b, r):  # bit-exact copy of the survivor's resolved state
        assert (other["x"].view("int32") == a["x"].view("int32")).all()
        assert other["mk"] == [(10, 0)] * 3
    # detected within the heartbeat timeout (+ scheduling slack)
    assert 0 < a["t_detect"] - a["crash"] < 5.0
    del store
