"""Replica recovery between two PROCESSES on one GPU (gloo for the small
host-side exchanges), so a single-GPU box runs the multi-process transfer
paths end to end: CUDA-IPC export/import of the replacement's buffers, the
copy-engine chain with stream-ordered epoch counters
(recovery.recover_replication_chain) and the fused undo + push kernel
(rw_undo_and_push, recovery.recover_replication_fused), and parallel replay
with the copy-engine ordered merge (replay.recover_parallel, merge.
CopyEngineMerger).  The replacement must receive the survivor's resolved
state bit for bit (copy semantics) and its markers; the survivor's
own state must equal an independent local apply_resolution;
parallel replay over the two helpers must equal the sequential replay and
the ghost run bit for bit, and so must the stage-per-worker
sub-pipeline (subpipeline.recover_subpipeline, 1F1B with copy-engine stage
boundaries).  The NCCL transfers need one device per rank
and are covered by tests/test_multigpu.py on boxes with >= 2 GPUs.
"""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SIZES = [100_003, 64, 2_000_017, 7, 1_234_567, 4096]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entry(transfer, rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _scenario(transfer, rank)))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
    finally:
        dist.destroy_process_group()


def _parallel(rank):
    from paper_2302_06173_b200 import ADAM, OptimizerHyper
    from paper_2302_06173_b200.recovery import release_peer_mappings
    from paper_2302_06173_b200.replay import BoundaryLog, Pipeline, Stage, recover_parallel, replay_group
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    ghost = Pipeline(p=4, dim=64, hidden=96, layers=2, rows=96, micro_batches=5, seed=4, kind=ADAM, hyper=h)
    log = BoundaryLog()
    for it in range(3):
        if it == 1:
            snaps = [ghost.stages[s].snapshot() for s in (1, 2)]
        ghost.run_iteration(log_group=(1, 2), log=log)
    seq = [Stage(s, 64, 96, 64, 2, 4, ADAM) for s in (1, 2)]
    par = [Stage(s, 64, 96, 64, 2, 4, ADAM) for s in (1, 2)]
    for a, b, sn in zip(seq, par, snaps):
        a.restore(sn)
        b.restore(sn)
    replay_group(seq, log, 1, 3, 96, 5, 4, h, first=False, last=False, dim=64)
    recover_parallel(par, log, 1, 3, 96, 5, 4, h, first=False, last=False, dim=64, rank=rank, d=2,
                     merge="copy_engine")
    torch.cuda.synchronize()
    out = dict(eq_seq=all(torch.equal(getattr(p.state, n), getattr(q.state, n))
                          for p, q in zip(par, seq) for n in ("x", "m", "v")),
               eq_ghost=all(torch.equal(getattr(p.state, n), getattr(ghost.stages[s].state, n))
                            for p, s in zip(par, (1, 2)) for n in ("x", "m", "v")))
    import torch.distributed as dist
    dist.barrier()
    release_peer_mappings()
    return out


def _subpipeline(rank):
    """Replay way (i): the group's stages folded onto the two workers, 1F1B,
    copy-engine boundaries with stream value-waits across the processes."""
    from paper_2302_06173_b200 import ADAM, OptimizerHyper
    from paper_2302_06173_b200.recovery import release_peer_mappings
    from paper_2302_06173_b200.replay import BoundaryLog, Pipeline, Stage
    from paper_2302_06173_b200.subpipeline import SubPipeline, recover_subpipeline, split_stages
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    g = Pipeline(p=6, dim=64, hidden=96, layers=2, rows=96, micro_batches=4, seed=8, kind=ADAM, hyper=h)
    log = BoundaryLog()
    ids = [1, 2, 3, 4]
    for it in range(3):
        if it == 1:
            snaps = {s: g.stages[s].snapshot() for s in ids}
        g.run_iteration(log_group=(1, 4), log=log)
    mine = [ids[i] for i in split_stages(len(ids), 2, rank)]
    sts = [Stage(s, 64, 96, 64, 2, 8, ADAM) for s in mine]
    for st, s in zip(sts, mine):
        st.restore(snaps[s])
    pipe = SubPipeline(sts, 4, 96, 64)
    recover_subpipeline(pipe, log, 1, 3, 8, h, first=False, last=False)
    torch.cuda.synchronize()
    ok = all(torch.equal(getattr(st.state, n), getattr(g.stages[s].state, n))
             for st, s in zip(sts, mine) for n in ("x", "m", "v"))
    import torch.distributed as dist
    dist.barrier()
    release_peer_mappings()
    return dict(eq_seq=ok, eq_ghost=ok)


def _scenario(transfer, rank):
    import torch.distributed as dist
    if transfer == "parallel":
        return _parallel(rank)
    if transfer == "subpipeline":
        return _subpipeline(rank)

    from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper, seeded_fill_
    from paper_2302_06173_b200.recovery import (apply_resolution, recover_replication_chain,
                                                recover_replication_fused, release_peer_mappings, resolve)
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    st = DeviceState(SIZES, kind=ADAM)
    twin = None
    if rank == 0:  # the survivor, torn after 3 of 6 groups
        for i, t in enumerate((st.x, st.g, st.m, st.v)):
            seeded_fill_(t, 40 + i)
        st.v.abs_()
        st.write_markers([(6, 0)] * len(SIZES))
        st.step(h, stop_after=3)
        twin = DeviceState(SIZES, kind=ADAM)
        for n in ("x", "g", "m", "v"):
            getattr(twin, n).copy_(getattr(st, n))
        twin.write_markers(st.markers())
    plan = resolve(st.markers() if rank == 0 else [], h, lens=SIZES if rank == 0 else None)
    if rank == 0:
        apply_resolution(twin, h, plan)
    if transfer == "chain":
        recover_replication_chain(st, h, plan, src=0, pieces=4, split=2)
    else:
        recover_replication_fused(st, h, plan, src=0)
    torch.cuda.synchronize()
    # the replacement's groups travel to the survivor over gloo (host copies)
    got = {}
    for n in ("x", "m", "v"):
        buf = getattr(st, n).cpu()
        dist.broadcast(buf, src=1)
        got[n] = buf
    out = dict(strategy=plan.strategy, markers=st.markers())
    if rank == 0:
        out["local_ok"] = all(torch.equal(getattr(st, n).view(torch.int32), getattr(twin, n).view(torch.int32))
                              for n in ("x", "m", "v"))
        out["replica_ok"] = all(
            torch.equal(got[n][o:o + k].view(torch.int32), getattr(st, n)[o:o + k].cpu().view(torch.int32))
            for n in ("x", "m", "v") for o, k in zip(st.offsets, st.sizes))
        out["twin_markers"] = twin.markers()
    dist.barrier()
    release_peer_mappings()
    return out


@pytest.mark.parametrize("transfer", ["chain", "fused", "parallel", "subpipeline"])
def test_two_processes_one_gpu(transfer):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_entry, args=(transfer, r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    try:
        for _ in ps:
            r, v = q.get(timeout=240)
            res[r] = v
            if isinstance(v, dict) and "error" in v:
                raise AssertionError(f"rank {r} raised:\n{v['error']}")
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.exitcode is None:
                p.kill()
                p.join()
    a, b = res[0], res[1]
    if transfer in ("parallel", "subpipeline"):
        assert a["eq_seq"] and b["eq_seq"] and a["eq_ghost"] and b["eq_ghost"]
        return
    assert a["strategy"] == b["strategy"] == "Undo"
    assert a["local_ok"], "survivor's resolved state differs from a local apply_resolution"
    assert a["replica_ok"], "replacement did not receive the survivor's resolved state bit for bit"
    assert a["markers"] == b["markers"] == a["twin_markers"]
