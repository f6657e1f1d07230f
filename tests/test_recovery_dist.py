"""Host logic of the N>1 recovery path (resolver all-reduces + replica
broadcast) with world-size-2 gloo on CPU.  The orchestration code is the same
one bench.py runs over NCCL on the B200 box; only the tensors are host
tensors here (HostState mimics the DeviceState surface it touches)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2302_06173_b200 import ADAM, AMSGRAD, OptimizerHyper
from paper_2302_06173_b200.recovery import recover, recover_replication, resolve


class HostState:
    def __init__(self, sizes, seed=None):
        n = sum(sizes)
        self.sizes = list(sizes)
        self.offsets = [sum(sizes[:i]) for i in range(len(sizes))]
        self.num_groups = len(sizes)
        self.device = torch.device("cpu")
        g = torch.Generator().manual_seed(seed or 0)
        mk = (lambda: torch.randn(n, generator=g)) if seed is not None else (lambda: torch.zeros(n))
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


def _to_wire(obj):
    """Tensors leave a worker as numpy arrays: a torch queue shares tensors by
    file descriptor, and the worker may exit before the parent receives."""
    if isinstance(obj, torch.Tensor):
        return ("__tensor__", obj.detach().cpu().numpy().copy())
    if isinstance(obj, dict):
        return {k: _to_wire(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return type(obj)(_to_wire(v) for v in obj)
    return obj


def _from_wire(obj):
    if isinstance(obj, tuple) and len(obj) == 2 and obj[0] == "__tensor__":
        return torch.from_numpy(obj[1])
    if isinstance(obj, dict):
        return {k: _from_wire(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return type(obj)(_from_wire(v) for v in obj)
    return obj


def _worker(rank, world, port, scenario, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = scenario(rank)
        q.put((rank, _to_wire(out)))
    finally:
        dist.destroy_process_group()


def _run(scenario, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {r: _from_wire(o) for r, o in (q.get(timeout=120) for _ in ps)}
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def scen_survivor_and_replacement(rank):
    h = OptimizerHyper(kind=ADAM)
    if rank == 0:  # survivor crashed mid-update: layers 1,2 updated (reverse order)
        mk = [(10, 0), (11, 1), (11, 1)]
        plan = resolve(mk, h, lens=[5, 5, 5])
        st = HostState([5, 5, 5], seed=3)
        st.write_markers([(10, 0), (10, 0), (10, 0)])  # after apply_resolution
    else:          # replacement: no state, joins the consensus with nothing
        plan = resolve([], h)
        st = HostState([5, 5, 5])
    nbytes = recover_replication(st, src=0)
    return dict(strategy=plan.strategy, target=plan.target, undo=plan.undo_ids,
                x=st.x.clone(), m=st.m.clone(), v=st.v.clone(), mk=st.markers(), nbytes=nbytes)


def test_replication_recovery_world2():
    res = _run(scen_survivor_and_replacement)
    a, b = res[0], res[1]
    assert a["strategy"] == b["strategy"] == "Undo"
    assert a["target"] == b["target"] == 10
    assert a["undo"] == [1, 2] and b["undo"] == []
    for k in ("x", "m", "v"):  # bit-exact copy semantics
        assert torch.equal(a[k].view(torch.int32), b[k].view(torch.int32))
    assert b["mk"] == [(10, 0)] * 3
    assert a["nbytes"] == 3 * 15 * 4


def scen_two_survivors_redo(rank):
    h = OptimizerHyper(kind=ADAM)
    # rank 0 updated 2 of 3 groups, rank 1 updated 1 of 3; gradients landed everywhere
    mk = [[(5, 0), (6, 1), (6, 1)], [(5, 0), (5, 0), (6, 1)]][rank]
    plan_min = resolve(mk, h, lens=[100, 100, 100], grad_ready=[True] * 3, policy="min_cost")
    plan_undo = resolve(mk, h, lens=[100, 100, 100], grad_ready=[True] * 3, policy="undo")
    plan_blocked = resolve(mk, h, lens=[100, 100, 100], grad_ready=[False] * 3, policy="min_cost")
    plan_ams = resolve(mk, OptimizerHyper(kind=AMSGRAD), lens=[100, 100, 100],
                       grad_ready=[True] * 3)
    return dict(min=(plan_min.strategy, plan_min.target, plan_min.actions),
                undo=(plan_undo.strategy, plan_undo.target, plan_undo.actions),
                blocked=plan_blocked.strategy, ams=(plan_ams.strategy, plan_ams.target))


def test_resolver_two_survivors_world2():
    res = _run(scen_two_survivors_redo)
    # max over ranks: undo cost = 200 elems (rank 0), redo cost = 200 (rank 1) -> tie -> undo
    assert res[0]["min"][0] == "Undo" and res[0]["min"][1] == 5
    assert res[0]["undo"] == ("Undo", 5, [0, 1, 1]) and res[1]["undo"] == ("Undo", 5, [0, 0, 1])
    assert res[0]["blocked"] == "Undo"
    # AMSGrad cannot undo but every lagging group holds its gradient -> redo to 6
    assert res[0]["ams"] == ("Redo", 6) and res[1]["ams"] == ("Redo", 6)


def scen_scatter_allgather(rank):
    """N >= 3: one survivor, two replacements, scatter + all-gather transfer
    (ragged length so the tail path runs too)."""
    h = OptimizerHyper(kind=ADAM)
    sizes = [5, 7, 11]
    if rank == 0:
        plan = resolve([(10, 0)] * 3, h, lens=sizes)
        st = HostState(sizes, seed=9)
        st.write_markers([(10, 0)] * 3)
    else:
        plan = resolve([], h)
        st = HostState(sizes)
    used, nbytes = recover(st, h, plan, src=0, transfer="scatter_allgather")
    return dict(used=used, x=st.x.clone(), m=st.m.clone(), v=st.v.clone(), mk=st.markers(), nbytes=nbytes)


def test_scatter_allgather_world3():
    res = _run(scen_scatter_allgather, world=3)
    for r in (1, 2):
        for k in ("x", "m", "v"):
            assert torch.equal(res[0][k].view(torch.int32), res[r][k].view(torch.int32))
        assert res[r]["mk"] == [(10, 0)] * 3
    assert all(res[r]["used"] == "scatter_allgather" for r in range(3))


def scen_pipelined(rank):
    """The pipelined transfer's run split and per-run broadcasts (no undo:
    consistent markers) over gloo, world 3."""
    h = OptimizerHyper(kind=ADAM)
    sizes = [5, 7, 11, 3, 13, 2]
    if rank == 0:
        st = HostState(sizes, seed=21)
        st.write_markers([(4, 0)] * len(sizes))
        plan = resolve(st.markers(), h, lens=sizes)
    else:
        st = HostState(sizes)
        plan = resolve([], h)
    used, nbytes = recover(st, h, plan, src=0, transfer="pipelined")
    return dict(used=used, strategy=plan.strategy, x=st.x.clone(), v=st.v.clone(), mk=st.markers(), nbytes=nbytes)


def test_pipelined_transfer_world3():
    res = _run(scen_pipelined, world=3)
    assert res[0]["strategy"] == "None"
    for r in (1, 2):
        assert torch.equal(res[r]["x"], res[0]["x"]) and torch.equal(res[r]["v"], res[0]["v"])
        assert res[r]["mk"] == [(4, 0)] * 6 and res[r]["used"] == "pipelined"
    assert res[0]["nbytes"] == 41 * 4 * 3


# ---- parallel recovery bookkeeping over gloo ----
def _oracle_sum(parts, out):
    """ordered_sum restated on the host (tensor.cpp:105-117: ((t0 + t1) + t2)
    + ..., one fp32 rounding per add) -- the oracle stands in for the device
    kernel so only the ownership / order / gather bookkeeping is under test."""
    import numpy as np
    acc = parts[0].numpy().astype(np.float32).copy()
    for p in parts[1:]:
        acc = (acc + p.numpy().astype(np.float32)).astype(np.float32)
    out.copy_(torch.from_numpy(acc))


def _mb_grad(mb, P):
    g = torch.Generator().manual_seed(1000 + mb)
    return torch.randn(P, generator=g) * (10.0 ** (mb % 3 - 1))  # mixed magnitudes: order matters


def scen_ordered_merge(rank):
    from paper_2302_06173_b200.replay import ordered_merge_finish, ordered_merge_start, parallel_assignment
    world = dist.get_world_size()
    out = {}
    for P, m in ((1000, 4), (77, 5), (130, 1), (5, 3)):  # ragged P: empty / short shards; helpers without mbs
        mine = parallel_assignment(m, world)[rank]
        bufs = {mb: _mb_grad(mb, P) for mb in mine}
        h = ordered_merge_start(bufs, P, m, device=torch.device("cpu"))
        out[(P, m)] = (ordered_merge_finish(h, summer=_oracle_sum), mine)
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_ordered_merge_bookkeeping_gloo(world):
    """Every helper ends with the ascending-mb ordered sum of ALL micro-batches'
    gradients, bit for bit equal to the sequential sum, and helper h owned
    exactly {mb : mb mod d == h} (Fig 6: {0,2} / {1,3})."""
    import numpy as np
    res = _run(scen_ordered_merge, world=world)
    for (P, m), _ in res[0].items():
        exp = _mb_grad(0, P).numpy().astype(np.float32)
        for mb in range(1, m):
            exp = (exp + _mb_grad(mb, P).numpy().astype(np.float32)).astype(np.float32)
        owned = sorted(mb for r in range(world) for mb in res[r][(P, m)][1])
        assert owned == list(range(m))
        for r in range(world):
            got, mine = res[r][(P, m)]
            assert mine == [mb for mb in range(m) if mb % world == r]
            assert np.array_equal(got.numpy().view(np.uint32), exp.view(np.uint32)), (P, m, r)
    if world == 2:
        assert res[0][(1000, 4)][1] == [0, 2] and res[1][(1000, 4)][1] == [1, 3]
