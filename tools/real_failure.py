"""End-to-end recovery from a REAL process crash on the B200 box (2 GPUs):

  rank 0 (survivor) and rank 1 train data-parallel replicas of an Adam state;
  both are in the middle of the layer-wise update (MidUpdate(G/2)) when rank 1
  dies (os._exit).  Rank 0 detects it from its stopped heartbeat, aborts the
  NCCL communicator, publishes the repair plan; a fresh replacement process
  claims rank 1's slot on the freed GPU; both join generation 1 over NCCL;
  then resolve + recover (the undo pipelined with the NCCL transfer) hands the
  replacement the resolved state, checked by device CRC32 of every buffer.

Prints one JSON line: detection, repair and recovery times (ms).
  python tools/real_failure.py [gpt2xl|small]
"""
import json
import os
import socket
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _sizes(which):
    from paper_2302_06173_b200.workloads import gpt2_xl_sizes
    return gpt2_xl_sizes() if which == "gpt2xl" else [4096 * 37 + 13] * 24


def _crcs(st):
    """CRC32 of each buffer's group contents (inter-group padding excluded)."""
    from paper_2302_06173_b200.logstore import crc32_device
    out = []
    for n in ("x", "m", "v"):
        packed = torch.cat([st.view(n, i) for i in range(st.num_groups)])
        out.append(crc32_device(packed.view(torch.uint8)))
    return out


def member(rank, port, which, q):
    from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper, seeded_fill_
    from paper_2302_06173_b200.membership import Membership, RepairPlan, abort_group, join_generation
    from paper_2302_06173_b200.recovery import prepare_transfer, recover, resolve
    import datetime
    torch.cuda.set_device(rank)
    store = dist.TCPStore("127.0.0.1", port, is_master=False, timeout=datetime.timedelta(seconds=120))
    join_generation(store, RepairPlan(0, 2, []), rank, "nccl", device_id=torch.device("cuda", rank))
    sizes = _sizes(which)
    st = DeviceState(sizes, kind=ADAM)
    for i, n in enumerate(("x", "g", "m", "v")):
        seeded_fill_(getattr(st, n), 2302 + i)   # identical replicas (same seeds on every rank)
    st.v.abs_()
    h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
    st.write_markers([(10, 0)] * st.num_groups)
    dist.barrier()
    mem = Membership(store, rank, 2, generation=0, interval=0.02, timeout=0.3)
    dist.barrier()
    st.step(h, stop_after=st.num_groups // 2)   # both replicas torn mid-update
    torch.cuda.synchronize()
    if rank == 1:
        store.set("crash_time", repr(time.time()))
        os._exit(1)
    mem.wait_failure(timeout=60)
    t_det = time.time()
    abort_group()
    plan = mem.publish_plan(settle=0.05)
    mem.stop()
    join_generation(store, plan, rank, "nccl", device_id=torch.device("cuda", rank))
    dist.all_reduce(torch.zeros(1, device="cuda"))  # connect the new communicator
    prepare_transfer(st)                            # and the transfer's per-buffer communicators
    torch.cuda.synchronize()
    t_join = time.time()
    p = resolve(st.markers(), h, lens=sizes)
    used, nbytes = recover(st, h, p, src=0)
    torch.cuda.synchronize()
    t_rec = time.time()
    crash = float(store.get("crash_time"))
    q.put(("survivor", dict(detect_ms=(mem.detected_at - crash) * 1e3,
                            repair_ms=(t_join - t_det) * 1e3,  # abort + plan + replacement joins + connect
                            recovery_ms=(t_rec - t_join) * 1e3, total_ms=(t_rec - crash) * 1e3,
                            strategy=p.strategy, undo_groups=len(p.undo_ids), transfer=used, bytes=nbytes,
                            crcs=_crcs(st), markers=st.markers()[:3])))
    dist.destroy_process_group()


def replacement(port, which, q):
    from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper
    from paper_2302_06173_b200.membership import claim_slot, join_generation
    from paper_2302_06173_b200.recovery import prepare_transfer, recover, resolve
    import datetime
    store = dist.TCPStore("127.0.0.1", port, is_master=False, timeout=datetime.timedelta(seconds=120))
    sizes = _sizes(which)
    # hot spare: the replica buffers are allocated on the spare GPU before any
    # failure (the spare of a real job has its own GPU; here it is the one the
    # crashed rank frees, so the allocation waits for the slot)
    plan, rank = claim_slot(store, 0, timeout=120)
    torch.cuda.set_device(rank)
    st = DeviceState(sizes, kind=ADAM)
    h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
    join_generation(store, plan, rank, "nccl", device_id=torch.device("cuda", rank))
    dist.all_reduce(torch.zeros(1, device="cuda"))
    prepare_transfer(st)
    p = resolve([], h)
    used, nbytes = recover(st, h, p, src=0)
    torch.cuda.synchronize()
    q.put(("replacement", dict(rank=rank, crcs=_crcs(st), markers=st.markers()[:3], transfer=used)))
    dist.destroy_process_group()


def main(which="small"):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    store = dist.TCPStore("127.0.0.1", port, is_master=True, wait_for_workers=False)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=member, args=(r, port, which, q)) for r in range(2)]
    for p in ps:
        p.start()
    rp = ctx.Process(target=replacement, args=(port, which, q))
    rp.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in ps + [rp]:
        p.join(timeout=120)
    sv, rep = res["survivor"], res["replacement"]
    out = dict(workload=which, crashed_rank_exit=ps[1].exitcode, replacement_rank=rep["rank"],
               identical=sv["crcs"] == rep["crcs"] and sv["markers"] == rep["markers"],
               **{k: (round(v, 2) if isinstance(v, float) else v) for k, v in sv.items() if k != "crcs"})
    print(json.dumps(out), flush=True)
    del store
    return out


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
