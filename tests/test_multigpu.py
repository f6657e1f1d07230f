"""Multi-GPU recovery on the B200 box (needs >= 2 GPUs; skipped otherwise).

* fused undo + NVLink push (rw_undo_and_push) == local undo, and the
  replacement receives a bit-exact copy (copy semantics);
* NCCL broadcast path gives the same bits;
* parallel replay over 2 ranks (scatter + ordered merge + all-gather) ==
  sequential replay bit for bit.
"""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

needs2 = pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                            reason="needs 2 GPUs")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_entry, args=(fn, r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    try:
        for _ in ps:
            r, v = q.get(timeout=240)
            out[r] = v
            if isinstance(v, dict) and "error" in v:  # fail fast: a peer may be blocked on this rank
                raise AssertionError(f"rank {r} raised:\n{v['error']}")
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.exitcode is None:  # our own child, stuck behind a failed peer
                p.kill()
                p.join()
    assert all(p.exitcode == 0 for p in ps)
    return out


def _entry(fn, rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        q.put((rank, fn(rank, world)))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
        raise
    finally:
        dist.destroy_process_group()


def scen_fused(rank, world):
    import torch.distributed as dist

    from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper, seeded_fill_
    from paper_2302_06173_b200.recovery import (apply_resolution, recover_replication,
                                                recover_replication_fused, resolve)
    sizes = [100_003, 64, 5_000_017, 7, 1_234_567, 4096]
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    st = DeviceState(sizes, kind=ADAM)
    if rank == 0:
        for i, t in enumerate((st.x, st.g, st.m, st.v)):
            seeded_fill_(t, 40 + i)
        st.v.abs_()
        st.write_markers([(6, 0)] * len(sizes))
        st.step(h, stop_after=3)                  # crash mid-update: groups 5,4,3 stepped
        plan = resolve(st.markers(), h, lens=sizes)
        # independent local resolution for comparison
        twin = DeviceState(sizes, kind=ADAM)
        for n in ("x", "g", "m", "v"):
            getattr(twin, n).copy_(getattr(st, n))
        twin.write_markers(st.markers())
        apply_resolution(twin, h, plan)
    else:
        plan = resolve([], h)
    nb = recover_replication_fused(st, h, plan, src=0)
    res = {n: getattr(st, n).clone() for n in ("x", "m", "v")}
    ok_local = True
    if rank == 0:
        ok_local = all(torch.equal(res[n].view(torch.int32), getattr(twin, n).view(torch.int32))
                       for n in ("x", "m", "v"))
    # bring rank 1's copy to rank 0 for comparison
    # (group contents only: the push moves every group; inter-group padding is not state)
    same = []
    for n in ("x", "m", "v"):
        other = res[n].clone()
        dist.broadcast(other, src=1)
        same.append(all(torch.equal(other[o:o + k].view(torch.int32), res[n][o:o + k].view(torch.int32))
                        for o, k in zip(st.offsets, st.sizes)))
    # the NCCL path on the same state gives the same bits
    st2 = DeviceState(sizes, kind=ADAM)
    if rank == 0:
        for n in ("x", "m", "v"):
            getattr(st2, n).copy_(res[n])
        st2.write_markers(st.markers())
    recover_replication(st2, src=0)
    same_nccl = all(torch.equal(getattr(st2, n)[o:o + k].view(torch.int32), res[n][o:o + k].view(torch.int32))
                    for n in ("x", "m", "v") for o, k in zip(st.offsets, st.sizes))
    # the pipelined path (undo run by run overlapped with async broadcasts) on a
    # fresh torn copy gives the same bits on both ranks
    from paper_2302_06173_b200.recovery import recover_replication_pipelined
    st3 = DeviceState(sizes, kind=ADAM)
    if rank == 0:
        for i, t in enumerate((st3.x, st3.g, st3.m, st3.v)):
            seeded_fill_(t, 40 + i)
        st3.v.abs_()
        st3.write_markers([(6, 0)] * len(sizes))
        st3.step(h, stop_after=3)
    recover_replication_pipelined(st3, h, plan, src=0, pieces=3)
    same_pipe = all(torch.equal(getattr(st3, n)[o:o + k].view(torch.int32), res[n][o:o + k].view(torch.int32))
                    for n in ("x", "m", "v") for o, k in zip(st.offsets, st.sizes))
    same_pipe = same_pipe and st3.markers() == st.markers()
    diffs = {}
    if rank == 0:
        for n in ("x", "m", "v"):
            d = (res[n] - getattr(twin, n)).abs()
            bad = torch.nonzero(res[n].view(torch.int32) != getattr(twin, n).view(torch.int32))
            diffs[n] = (float(d.max()), int(bad.numel()), bad[:5].flatten().tolist())
    return dict(strategy=plan.strategy, ok_local=ok_local, same=all(same), same_list=same,
                same_nccl=same_nccl, same_pipe=same_pipe, markers=st.markers(), nbytes=nb, diffs=diffs)


@needs2
def test_fused_undo_push_bitexact():
    out = _run(scen_fused)
    print(out[0]["diffs"], out[0]["same_list"], out[1]["same_list"], out[0]["same_nccl"], out[0]["markers"])
    assert out[0]["strategy"] == "Undo"
    assert out[0]["ok_local"]
    assert out[0]["same"] and out[1]["same"]
    assert out[0]["same_nccl"] and out[1]["same_nccl"]
    assert out[0]["same_pipe"] and out[1]["same_pipe"]
    assert out[0]["markers"] == out[1]["markers"] == [(6, 0)] * 6


def scen_parallel_replay(rank, world):
    import torch.distributed as dist

    from paper_2302_06173_b200 import ADAM, OptimizerHyper
    from paper_2302_06173_b200.replay import (BoundaryLog, Pipeline, Stage, recover_parallel,
                                              replay_group)
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    ghost = Pipeline(p=3, dim=64, hidden=128, layers=2, rows=128, micro_batches=4, seed=11, kind=ADAM, hyper=h)
    log = BoundaryLog()
    for it in range(3):
        if it == 1:
            snap = ghost.stages[1].snapshot()
        ghost.run_iteration(log_group=(1, 1), log=log)
    seq = Stage(1, 64, 128, 64, 2, 11, ADAM)
    seq.restore(snap)
    replay_group([seq], log, 1, 3, 128, 4, 11, h, first=False, last=False, dim=64)
    par = Stage(1, 64, 128, 64, 2, 11, ADAM)
    par.restore(snap)
    recover_parallel([par], log, 1, 3, 128, 4, 11, h, first=False, last=False, dim=64, rank=rank, d=world)
    res = dict(eq_seq=all(torch.equal(getattr(par.state, n), getattr(seq.state, n)) for n in ("x", "m", "v")),
               eq_ghost=torch.equal(par.state.x, ghost.stages[1].state.x))
    # a 3-stage middle group, odd micro-batch count (uneven helpers), merges
    # overlapped with the backward of the earlier stages
    g5 = Pipeline(p=5, dim=64, hidden=96, layers=2, rows=96, micro_batches=5, seed=4, kind=ADAM, hyper=h)
    log5 = BoundaryLog()
    for it in range(3):
        if it == 1:
            snaps = [g5.stages[s].snapshot() for s in (1, 2, 3)]
        g5.run_iteration(log_group=(1, 3), log=log5)
    grp = [Stage(s, 64, 96, 64, 2, 4, ADAM) for s in (1, 2, 3)]
    for st, sn in zip(grp, snaps):
        st.restore(sn)
    recover_parallel(grp, log5, 1, 3, 96, 5, 4, h, first=False, last=False, dim=64, rank=rank, d=world)
    res["eq_group"] = all(torch.equal(getattr(grp[k].state, n), getattr(g5.stages[s].state, n))
                          for k, s in enumerate((1, 2, 3)) for n in ("x", "m", "v"))
    return res


WORLD = min(4, torch.cuda.device_count()) if torch.cuda.is_available() else 0


@needs2
def test_parallel_replay_bitexact():
    """All visible GPUs (up to 4) as helpers."""
    out = _run(scen_parallel_replay, world=WORLD)
    for r in range(WORLD):
        assert out[r]["eq_seq"] and out[r]["eq_ghost"]
        assert out[r]["eq_group"]


@needs2
def test_two_devices_in_one_process():
    """Per-device kernel attributes: the fused kernels, the CRC and the GEMMs
    launched on cuda:0 and then on cuda:1 from the same process."""
    from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper, seeded_fill_
    from paper_2302_06173_b200.logstore import crc32_device
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    outs = []
    for d in (0, 1):
        with torch.cuda.device(d):
            st = DeviceState([70_001, 3_000], kind=ADAM, device=d)
            for i, n in enumerate(("x", "g", "m", "v")):
                seeded_fill_(getattr(st, n), 5 + i)
            st.v.abs_()
            st.step(h)
            st.undo(h)
            st.check_finite()
            outs.append((st.x.cpu(), crc32_device(st.x.view(torch.uint8))))
            from paper_2302_06173_b200.replay import Stage
            sg = Stage(0, 64, 128, 64, 2, 3, ADAM, device=d)
            acts = sg.new_acts(128)
            acts[0].normal_()
            sg.forward(acts)
            torch.cuda.synchronize(d)
    assert torch.equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]


def scen_subpipeline(rank, world):
    """Replay way (i): the failed group's stages folded onto the GPUs (1F1B,
    copy-engine boundaries) == the ghost run bit for bit, for a middle group
    and for a group ending at the loss."""
    from paper_2302_06173_b200 import ADAM, OptimizerHyper
    from paper_2302_06173_b200.replay import BoundaryLog, Pipeline, Stage
    from paper_2302_06173_b200.subpipeline import SubPipeline, one_f_one_b, recover_subpipeline, split_stages
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    res = {"sched": one_f_one_b(2, 4, rank)}
    # 4-stage groups of a 7-stage pipeline: 2 stages per GPU at d=2, 1 at d=4
    for name, grp, last in (("middle", (1, 4), False), ("tail", (3, 6), True)):
        g = Pipeline(p=7, dim=64, hidden=96, layers=2, rows=96, micro_batches=4, seed=8, kind=ADAM, hyper=h)
        log = BoundaryLog()
        ids = list(range(grp[0], grp[1] + 1))
        for it in range(3):
            if it == 1:
                snaps = {s: g.stages[s].snapshot() for s in ids}
            g.run_iteration(log_group=grp, log=log)
        mine = [ids[i] for i in split_stages(len(ids), world, rank)]
        sts = [Stage(s, 64, 96, 64, 2, 8, ADAM) for s in mine]
        for st, s in zip(sts, mine):
            st.restore(snaps[s])
        pipe = SubPipeline(sts, 4, 96, 64)
        recover_subpipeline(pipe, log, 1, 3, 8, h, first=False, last=last)
        res[name] = all(torch.equal(getattr(st.state, n), getattr(g.stages[s].state, n))
                        for st, s in zip(sts, mine) for n in ("x", "m", "v"))
    return res


@needs2
def test_subpipeline_replay_bitexact():
    """All visible GPUs (up to 4) as pipeline workers."""
    out = _run(scen_subpipeline, world=WORLD)
    assert out[0]["sched"] == [("F", 0), ("F", 1), ("B", 0), ("F", 2), ("B", 1), ("F", 3), ("B", 2), ("B", 3)]
    assert out[1]["sched"] == [("F", 0), ("B", 0), ("F", 1), ("B", 1), ("F", 2), ("B", 2), ("F", 3), ("B", 3)]
    for r in range(WORLD):
        assert out[r]["middle"] and out[r]["tail"], out[r]


def scen_recovery_all(rank, world):
    """Replica recovery to every other rank (1 survivor, world-1 replacements):
    pipelined (undo overlapped with per-buffer NCCL broadcasts) and
    undo-then-broadcast give every rank the survivor's resolved bits."""
    import torch.distributed as dist

    from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper, seeded_fill_
    from paper_2302_06173_b200.logstore import crc32_device
    from paper_2302_06173_b200.recovery import recover, resolve
    sizes = [100_003, 64, 2_000_017, 7, 1_234_567, 4096, 77]
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    out = {}
    for transfer in ("pipelined", "broadcast", "chain"):
        st = DeviceState(sizes, kind=ADAM)
        if rank == 0:
            for i, t in enumerate((st.x, st.g, st.m, st.v)):
                seeded_fill_(t, 50 + i)
            st.v.abs_()
            st.write_markers([(9, 0)] * len(sizes))
            st.step(h, stop_after=4)
        plan = resolve(st.markers() if rank == 0 else [], h, lens=sizes if rank == 0 else None)
        used, _ = recover(st, h, plan, src=0, transfer=transfer)
        crc = [crc32_device(torch.cat([st.view(n, i) for i in range(len(sizes))]).view(torch.uint8))
               for n in ("x", "m", "v")]
        allc = [None] * world
        dist.all_gather_object(allc, (crc, st.markers()))
        out[transfer] = dict(used=used, same=all(c == allc[0] for c in allc), strategy=plan.strategy,
                             markers=st.markers())
    return out


@needs2
def test_recovery_to_all_ranks_bitexact():
    out = _run(scen_recovery_all, world=WORLD)
    for r in range(WORLD):
        for tr in ("pipelined", "broadcast", "chain"):
            assert out[r][tr]["same"] and out[r][tr]["strategy"] == "Undo", (r, tr, out[r][tr])
            assert out[r][tr]["markers"] == [(9, 0)] * 7


def scen_lamb_recovery(rank, world):
    """LAMB (saved trust ratios) through the chain and pipelined transfers:
    the replacement gets the survivor's state AND its trust-ratio stacks, so a
    later undo on the replacement matches the survivor's bit for bit."""
    import torch.distributed as dist

    from paper_2302_06173_b200 import LAMB, DeviceState, OptimizerHyper, seeded_fill_
    from paper_2302_06173_b200.recovery import recover, resolve
    sizes = [50_001, 4096, 777, 300_000]
    h = OptimizerHyper(kind=LAMB, lr=1e-3, weight_decay=0.01)
    out = {}
    for transfer in ("chain", "pipelined"):
        st = DeviceState(sizes, kind=LAMB)
        if rank == 0:
            for i, t in enumerate((st.x, st.g, st.m, st.v)):
                seeded_fill_(t, 70 + i)
            st.v.abs_()
            st.write_markers([(4, 0)] * len(sizes))
            st.step(h)                 # a completed LAMB step (ratios saved) ...
            st.clear_updated()
            st.step(h, stop_after=2)   # ... then a torn one
        plan = resolve(st.markers() if rank == 0 else [], h, lens=sizes if rank == 0 else None)
        recover(st, h, plan, src=0, transfer=transfer)
        # everyone undoes the completed step with its (replicated) saved ratio
        st.write_markers([(5, 1)] * len(sizes))
        st.undo(h)
        x = st.x.clone()
        allx = [torch.empty_like(x) for _ in range(world)]
        dist.all_gather(allx, x)
        out[transfer] = dict(strategy=plan.strategy,
                             same=all(torch.equal(a[o:o + n], allx[0][o:o + n]) for a in allx
                                      for o, n in zip(st.offsets, st.sizes)),
                             saved=[len(st.saved_scalars(i)) for i in range(len(sizes))])
    return out


@needs2
def test_lamb_recovery_replicates_saved_ratios():
    out = _run(scen_lamb_recovery, world=WORLD)
    for r in range(WORLD):
        for tr in ("chain", "pipelined"):
            assert out[r][tr]["strategy"] == "Undo" and out[r][tr]["same"], (r, tr, out[r][tr])
            assert out[r][tr]["saved"] == [0, 0, 0, 0]
