"""Recovery orchestration: consistency resolver + replica recovery.

Reference contracts (recovery.cpp is absent):
  * consensus_iteration  SPEC:475-483  (min over survivors)
  * apply_undo           SPEC:484-492  (undo blocks beyond the target)
  * recover_replication  SPEC:493-501  (bit-exact copy of the survivor state)

One process per GPU.  ``torch.distributed`` is the plumbing: NCCL over
NVLink on the B200 box (the MIN/MAX all-reduces of the resolver and the
ncclBroadcast of the resolved state), gloo in the CPU tests of the host
logic.  The per-group decisions are made by the C++ resolver
(csrc/resolver_planner.cpp) and the arithmetic by the fused CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field
from typing import Sequence

import torch
import torch.distributed as dist

from ._lib import (ACT_REDO, ACT_UNDO, LIB, POLICY_MIN_COST, POLICY_UNDO, STRATEGY_GLOBAL_ROLLBACK,
                   STRATEGY_NAMES, STRATEGY_REDO, STRATEGY_UNDO, RwError, check, rw_group, rw_hyper,
                   rw_resolve_summary)

U64_MAX = 2**64 - 1


@dataclass
class ResolvePlan:
    strategy: str
    target: int
    actions: list[int]                  # per local group: 0 none, 1 undo, 2 redo
    summary: dict = field(default_factory=dict)

    @property
    def undo_ids(self) -> list[int]:
        return [i for i, a in enumerate(self.actions) if a == ACT_UNDO]

    @property
    def redo_ids(self) -> list[int]:
        return [i for i, a in enumerate(self.actions) if a == ACT_REDO]


def _groups_from_markers(markers: Sequence[tuple[int, int]], lens: Sequence[int] | None = None):
    g = (rw_group * max(len(markers), 1))()
    for i, (t, u) in enumerate(markers):
        g[i].offset, g[i].len = 0, (lens[i] if lens is not None else 1)
        g[i].t, g[i].updated, g[i].flags = t, u, 0
    return g


def _allreduce_u64(vals: list[int], op, group=None, device=None) -> list[int]:
    """All-reduce a few uint64 counters (sent as int64; values < 2^63)."""
    if not (dist.is_available() and dist.is_initialized()):
        return list(vals)
    backend = dist.get_backend(group)
    if backend == "nccl":
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device("cpu")
    t = torch.tensor([int(v) for v in vals], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=op, group=group)
    return [int(v) for v in t.cpu().tolist()]


def resolve(markers: Sequence[tuple[int, int]], hyper, lens: Sequence[int] | None = None,
            grad_ready: Sequence[bool] | None = None, policy: str = "undo", group=None,
            device=None) -> ResolvePlan:
    """Consensus + per-group undo/redo decision across all survivor ranks.

    markers: this rank's (t, updated) per group (read from the device table).
    Exchanges: one MIN/MAX all-reduce of (t_min, t_max), one MAX all-reduce of
    the costs / blocks relative to the global t_min.
    """
    h: rw_hyper = hyper.to_c() if hasattr(hyper, "to_c") else hyper
    g = _groups_from_markers(markers, lens)
    n = len(markers)
    ready = None
    if grad_ready is not None:
        ready = (C.c_uint8 * max(n, 1))(*[1 if r else 0 for r in grad_ready])
    loc = rw_resolve_summary()
    check(LIB.rw_resolve_summarize(g, n, ready, C.byref(h), U64_MAX, C.byref(loc)))
    t_min = min(loc.t_min, U64_MAX >> 1)  # n == 0 -> UINT64_MAX (MIN identity), int64-safe
    lo = _allreduce_u64([t_min], dist.ReduceOp.MIN if dist.is_available() else None, group, device)[0]
    hi = _allreduce_u64([loc.t_max], dist.ReduceOp.MAX if dist.is_available() else None, group,
                        device)[0]
    s2 = rw_resolve_summary()
    check(LIB.rw_resolve_summarize(g, n, ready, C.byref(h), lo, C.byref(s2)))
    costs = _allreduce_u64([s2.undo_elems, s2.redo_elems, s2.redo_blocked, s2.undo_blocked],
                           dist.ReduceOp.MAX if dist.is_available() else None, group, device)
    glob = rw_resolve_summary()
    glob.t_min, glob.t_max = lo, hi
    glob.undo_elems, glob.redo_elems, glob.redo_blocked, glob.undo_blocked = costs
    acts = (C.c_uint8 * max(n, 1))()
    tgt, st = C.c_uint64(), C.c_int32()
    pol = POLICY_MIN_COST if policy == "min_cost" else POLICY_UNDO
    check(LIB.rw_resolve_plan(C.byref(glob), pol, g, n, acts, C.byref(tgt), C.byref(st)))
    return ResolvePlan(STRATEGY_NAMES[st.value], tgt.value, list(acts[:n]),
                       dict(t_min=lo, t_max=hi, undo_elems=costs[0], redo_elems=costs[1],
                            redo_blocked=costs[2], undo_blocked=costs[3]))


def apply_resolution(state, hyper, plan: ResolvePlan, grad: torch.Tensor | None = None,
                     stream=None) -> None:
    """Execute a ResolvePlan on a DeviceState with the fused kernels.

    Undo: groups beyond the target whose updated flag was already cleared
    (completed iteration) are re-armed first — the spec gap of SURVEY §8a
    row a13: the decision is on t, at most one step back, g still caches that
    step's gradient (one version kept).
    Redo: lagging groups are stepped with their synchronised gradient `grad`.
    """
    if plan.strategy == STRATEGY_NAMES[STRATEGY_GLOBAL_ROLLBACK]:
        raise RwError(101, "plan requires a global checkpoint rollback (SPEC:488)")
    if plan.strategy == STRATEGY_NAMES[STRATEGY_UNDO] and plan.undo_ids:
        undo = set(plan.undo_ids)
        mk = state.markers(stream)
        if any(mk[i][1] == 0 for i in undo):
            state.write_markers([(t, 1 if i in undo else u) for i, (t, u) in enumerate(mk)], stream)
        # undo in reverse update order (first layer's update was the last)
        order = [i for i in reversed(state.update_order()) if i in undo]
        state.undo(hyper, order, stream=stream)
    elif plan.strategy == STRATEGY_NAMES[STRATEGY_REDO] and plan.redo_ids:
        if grad is None:
            raise RwError(101, "redo needs the synchronised gradient buffer")
        redo = set(plan.redo_ids)
        order = [i for i in state.update_order() if i in redo]
        state.step(hyper, order, grad=grad, stream=stream)


_PEER_MAPS: dict[bytes, C.c_void_p] = {}  # IPC handle -> mapped base (kept for reuse)
LAST_FUSED_INFO: dict = {}


def release_peer_mappings() -> None:
    for base in _PEER_MAPS.values():
        LIB.rw_ipc_close(base)
    _PEER_MAPS.clear()


def _export(t: torch.Tensor) -> tuple[bytes, int]:
    h = (C.c_uint8 * 64)()
    off = C.c_uint64()
    check(LIB.rw_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off)))
    return bytes(h), off.value


def _allgather_exports(tensors: Sequence[torch.Tensor], group=None) -> list[list[tuple[bytes, int]]]:
    """Every rank's CUDA-IPC exports of `tensors` (the same count on every
    rank): the 64-byte handles and offsets travel as one small byte tensor in
    a single all_gather on the group's backend (~0.05 ms over NCCL) instead
    of a pickled all_gather_object (~1 ms)."""
    world = dist.get_world_size(group)
    k = len(tensors)
    rec = torch.empty(k, 72, dtype=torch.uint8)
    for i, t in enumerate(tensors):
        hb, off = _export(t)
        rec[i, :64] = torch.frombuffer(bytearray(hb), dtype=torch.uint8)
        rec[i, 64:] = torch.frombuffer(bytearray(int(off).to_bytes(8, "little")), dtype=torch.uint8)
    dev = tensors[0].device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = rec.to(dev)
    allr = torch.empty(world * k, 72, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(allr, mine, group=group)
    flat = allr.cpu().numpy()
    return [[(flat[r * k + i, :64].tobytes(), int.from_bytes(flat[r * k + i, 64:].tobytes(), "little"))
             for i in range(k)] for r in range(world)]


def recover_replication_fused(state, hyper, plan: ResolvePlan, src: int, include_grad: bool = False,
                              group=None, stream=None) -> int:
    """apply_undo + recover_replication in ONE kernel on the survivor `src`:
    the undo of plan.undo_ids is computed tile by tile and every resolved tile
    (and every untouched group) is written straight into each replacement's
    HBM over NVLink (CUDA IPC-mapped peer buffers, bulk stores from the same
    kernel) — the transfer hides the undo.  Replacements only publish their
    buffers and wait.  Returns bytes written per replacement."""
    if not (dist.is_available() and dist.is_initialized()):
        raise RwError(17, "NoReplica: no process group")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    names = ["x"] + (["g"] if include_grad else []) + [n for n in ("m", "v") if getattr(state, n) is not None]
    mine = None if rank == src else {n: _export(getattr(state, n)) for n in names}
    allh: list = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    nbytes = sum(getattr(state, n).numel() * getattr(state, n).element_size() for n in names)
    if rank == src:
        h = hyper.to_c() if hasattr(hyper, "to_c") else hyper
        sh = C.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
        undo = [i for i, a in enumerate(plan.actions) if a == ACT_UNDO] if plan.strategy == "Undo" else []
        if undo:  # the spec-gap re-arm of apply_resolution (decide on t, flag cleared at iteration end)
            mk = state.markers(stream)
            if any(mk[i][1] == 0 for i in undo):
                su = set(undo)
                state.write_markers([(t, 1 if i in su else u) for i, (t, u) in enumerate(mk)], stream)
        t0 = time.perf_counter()
        first = True
        peers = []
        for r in range(world):
            if r == src:
                continue
            peer = {}
            for n, (hb, off) in allh[r].items():
                if hb not in _PEER_MAPS:  # map each replacement allocation once
                    base = C.c_void_p()
                    check(LIB.rw_ipc_import(hb, C.byref(base)))
                    _PEER_MAPS[hb] = base
                peer[n] = C.c_void_p(_PEER_MAPS[hb].value + off)
            peers.append(peer)
        t1 = time.perf_counter()
        cs = stream or torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        for peer in peers:
            ids = undo if first else []  # later replacements receive the already-resolved state
            arr = (C.c_uint32 * max(len(ids), 1))(*ids)
            check(LIB.rw_undo_and_push(state.handle, C.byref(h), arr, len(ids), peer["x"], peer.get("g"),
                                       peer.get("m"), peer.get("v"), sh))
            first = False
        e1.record(cs)
        cs.synchronize()
        LAST_FUSED_INFO.clear()
        LAST_FUSED_INFO.update(map_ms=(t1 - t0) * 1e3, kernel_ms=e0.elapsed_time(e1))
    dist.barrier(group=group)
    _broadcast_saved_scalars(state, src, group)
    mk = state.markers()
    backend = dist.get_backend(group)
    dev = state.device if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([v for pair in mk for v in pair], dtype=torch.int64, device=dev)
    dist.broadcast(t, src=src, group=group)
    flat = t.cpu().tolist()
    state.write_markers([(flat[2 * i], flat[2 * i + 1]) for i in range(len(mk))])
    return nbytes


def _broadcast_saved_scalars(state, src: int, group=None) -> None:
    """LAMB: the replacement needs the survivor's trust-ratio stacks
    (ParamBlock::saved_scalars) for a later undo — one small broadcast."""
    from ._lib import LAMB
    from .optim import TRUST_DEPTH
    if getattr(state, "kind", None) != LAMB:
        return
    G = state.num_groups
    backend = dist.get_backend(group)
    dev = state.device if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(G, 1 + TRUST_DEPTH, dtype=torch.float64)
    if dist.get_rank(group) == src:
        for i in range(G):
            vals = state.saved_scalars(i)
            buf[i, 0] = len(vals)
            buf[i, 1:1 + len(vals)] = torch.tensor(vals, dtype=torch.float64)
    t = buf.to(dev)
    dist.broadcast(t, src=src, group=group)
    if dist.get_rank(group) != src:
        rows = t.cpu()
        for i in range(G):
            c = int(rows[i, 0])
            state.set_saved_scalars(i, rows[i, 1:1 + c].tolist())


def _scatter_allgather(buf: torch.Tensor, src: int, group=None) -> None:
    """Broadcast of `buf` from `src` as scatter + all-gather: the source hands
    slice r to rank r (its egress carries the state once), then every rank
    all-gathers the slices (in place; NCCL uses NVLS on NVSwitch), so each
    rank's ingress carries the state once and no single link is serialised
    over the replacements."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = buf.numel()
    chunk = n // world
    main = chunk * world
    if chunk:
        views = [buf[r * chunk:(r + 1) * chunk] for r in range(world)]
        glob = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)  # noqa: E731
        if rank == src:
            ops = [dist.P2POp(dist.isend, views[r], glob(r), group) for r in range(world) if r != src]
        else:
            ops = [dist.P2POp(dist.irecv, views[rank], glob(src), group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(buf[:main], views[rank], group=group)
        else:  # gloo: list form
            parts = [torch.empty_like(views[rank]) for _ in range(world)]
            dist.all_gather(parts, views[rank].clone(), group=group)
            for r in range(world):
                if r != rank:
                    views[r].copy_(parts[r])
    if main < n:  # the tail (< world elements)
        dist.broadcast(buf[main:], src=glob(src) if chunk else src, group=group)


def recover_replication(state, src: int, include_grad: bool = False, group=None,
                        algo: str = "broadcast") -> int:
    """recover_replication: copy the resolved state from the
    surviving rank `src` to every other rank of `group` (NCCL over NVLink):
    algo "broadcast" (ncclBroadcast) or "scatter_allgather" (each link carries
    the state once; measured slower than ncclBroadcast on the B200 box).
    Bit-exact copy semantics; markers travel with it.  Returns bytes received
    per replacement."""
    if not (dist.is_available() and dist.is_initialized()):
        raise RwError(17, "NoReplica: no process group")
    bufs = [state.x] + ([state.g] if include_grad else [])
    bufs += [b for b in (state.m, state.v) if b is not None]
    for b in bufs:
        if algo == "scatter_allgather":
            _scatter_allgather(b, src, group)
        else:
            dist.broadcast(b, src=src, group=group)
    _broadcast_saved_scalars(state, src, group)
    mk = state.markers()
    backend = dist.get_backend(group)
    dev = state.device if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([v for pair in mk for v in pair], dtype=torch.int64, device=dev)
    dist.broadcast(t, src=src, group=group)
    flat = t.cpu().tolist()
    state.write_markers([(flat[2 * i], flat[2 * i + 1]) for i in range(len(mk))])
    return sum(b.numel() * b.element_size() for b in bufs)


_BUFFER_COMMS: dict = {}


def _buffer_comms(k: int, group=None) -> list:
    """One communicator per state buffer (created once, collectively), so the
    broadcasts of x, m and v proceed concurrently instead of queueing on one
    NCCL stream.  With gloo (CPU tests) the given group is reused."""
    if dist.get_backend(group) != "nccl":
        return [group] * k
    key = (k, id(group))
    if key not in _BUFFER_COMMS:
        ranks = None if group is None else dist.get_process_group_ranks(group)
        _BUFFER_COMMS[key] = [dist.new_group(ranks=ranks, backend="nccl") for _ in range(k)]
    return _BUFFER_COMMS[key]


def prepare_transfer(state, include_grad: bool = False, group=None) -> None:
    """Create and connect the per-buffer communicators of the pipelined
    transfer and map every peer's state buffers for the copy-engine chain,
    ahead of time (collective): right after a repaired process group is
    formed, so the recovery itself pays neither NCCL initialisation nor CUDA
    IPC mapping."""
    names = ["x"] + (["g"] if include_grad else []) + [n for n in ("m", "v") if getattr(state, n) is not None]
    for cg in _buffer_comms(len(names), group):
        dev = state.device if dist.get_backend(cg) == "nccl" else torch.device("cpu")
        dist.all_reduce(torch.zeros(1, device=dev), group=cg)
    if dist.get_backend(group) == "nccl":  # and map every peer's buffers for the copy-engine chain
        mine = {n: _export(getattr(state, n)) for n in names}
        allh: list = [None] * dist.get_world_size(group)
        dist.all_gather_object(allh, mine, group=group)
        for r, h in enumerate(allh):
            if r == dist.get_rank(group):
                continue
            for hb, _ in h.values():
                if hb not in _PEER_MAPS:
                    base = C.c_void_p()
                    check(LIB.rw_ipc_import(hb, C.byref(base)))
                    _PEER_MAPS[hb] = base


def recover_replication_pipelined(state, hyper, plan: ResolvePlan, src: int, include_grad: bool = False,
                                  group=None, pieces: int = 4, lead: int = 0) -> int:
    """apply_undo + recover_replication as a two-stage pipeline over `pieces`
    contiguous runs of groups: the survivor undoes run i on its stream while
    NCCL broadcasts the already-resolved run i-1 (async broadcasts of buffer
    views; NCCL's kernels co-reside with the memory-bound undo kernel), so the
    undo hides behind the transfer for any number of replacements.  Every rank
    derives the same runs from the shared layout.  Returns bytes per
    replacement.  lead > 0 paces the survivor's undo: run i starts only once the
    broadcasts of run i - lead are done (an undo burst at full HBM bandwidth
    slows the transfers it overlaps)."""
    if not (dist.is_available() and dist.is_initialized()):
        raise RwError(17, "NoReplica: no process group")
    rank = dist.get_rank(group)
    names = ["x"] + (["g"] if include_grad else []) + [n for n in ("m", "v") if getattr(state, n) is not None]
    G = state.num_groups
    undo = set(plan.undo_ids) if plan.strategy == STRATEGY_NAMES[STRATEGY_UNDO] else set()
    if rank == src and plan.strategy not in (STRATEGY_NAMES[STRATEGY_UNDO], "None"):
        apply_resolution(state, hyper, plan)  # redo: step first, then copy
    if rank == src and undo:  # the re-arm of apply_resolution (decide on t)
        mk = state.markers()
        if any(mk[i][1] == 0 for i in undo):
            state.write_markers([(t, 1 if i in undo else u) for i, (t, u) in enumerate(mk)])
    total = sum(state.sizes)
    runs, start, acc = [], 0, 0
    for i, n in enumerate(state.sizes):  # contiguous runs of ~total/pieces elements
        acc += n
        if acc >= total * (len(runs) + 1) / pieces or i == G - 1:
            runs.append((start, i + 1))
            start = i + 1
    comms = _buffer_comms(len(names), group)  # x, m, v transfers run concurrently
    works = []
    for k, (g0, g1) in enumerate(runs):
        lo, hi = state.offsets[g0], state.offsets[g1 - 1] + state.sizes[g1 - 1]
        if rank == src:
            ids = [i for i in range(g0, g1) if i in undo]
            if ids:
                if lead and k >= lead:
                    for w in works[(k - lead) * len(names):(k - lead + 1) * len(names)]:
                        w.wait()  # stream-side: the current stream waits for those broadcasts
                state.undo(hyper, ids)
        for n, cg in zip(names, comms):
            gsrc = dist.get_global_rank(cg, src) if group is not None else src
            works.append(dist.broadcast(getattr(state, n)[lo:hi], src=gsrc, group=cg, async_op=True))
    for w in works:
        w.wait()
    _broadcast_saved_scalars(state, src, group)
    mk = state.markers()
    backend = dist.get_backend(group)
    dev = state.device if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([v for pair in mk for v in pair], dtype=torch.int64, device=dev)
    dist.broadcast(t, src=src, group=group)
    flat = t.cpu().tolist()
    state.write_markers([(flat[2 * i], flat[2 * i + 1]) for i in range(len(mk))])
    return sum(sum(state.sizes) * getattr(state, n).element_size() for n in names)


_CE_CHAINS: dict = {}
# (pieces, lead) of the pipelined transfer recover() uses; RW_PIPE="pieces,lead" overrides (sweeps)
_PIPE = tuple(int(v) for v in os.environ.get("RW_PIPE", "4,0").split(","))


def _runs_of(state, pieces: int) -> list[tuple[int, int]]:
    """Contiguous runs of groups of ~total/pieces elements (same on every rank)."""
    G, total = state.num_groups, sum(state.sizes)
    runs, start, acc = [], 0, 0
    for i, n in enumerate(state.sizes):
        acc += n
        if acc >= total * (len(runs) + 1) / pieces or i == G - 1:
            runs.append((start, i + 1))
            start = i + 1
    return runs


def recover_replication_chain(state, hyper, plan: ResolvePlan, src: int, include_grad: bool = False,
                              group=None, pieces: int = 16, split: int = 1) -> int:
    """apply_undo + recover_replication over the copy engines, as a pipelined
    chain: the survivor undoes run i of the groups while its DMA engines push
    the already-resolved run i-1 into the first replacement's HBM (CUDA IPC);
    each replacement forwards every run to the next one as soon as the run's
    epoch counter lands (cuStreamWaitValue64 -> cudaMemcpyAsync ->
    cuStreamWriteValue64, all stream-ordered, no kernel).  The copy engines
    write NVLink at ~780 GB/s against ~717 for SM stores (tools/peer_bw.cu),
    every link carries the state once, and the chain adds only one run's
    transfer per extra hop.  Returns bytes per replacement."""
    if not (dist.is_available() and dist.is_initialized()):
        raise RwError(17, "NoReplica: no process group")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    names = ["x"] + (["g"] if include_grad else []) + [n for n in ("m", "v") if getattr(state, n) is not None]
    runs = _runs_of(state, pieces)  # undo granularity (whole groups)
    # copy granularity: every run's element span in `split` equal sub-ranges
    # (copies need no group alignment), so each hop lags one sub-range only
    spans = []
    for g0, g1 in runs:
        lo, hi = state.offsets[g0], state.offsets[g1 - 1] + state.sizes[g1 - 1]
        step = -(-(hi - lo) // split)
        spans.append([(a, min(hi, a + step)) for a in range(lo, hi, step)])
    n_pieces = sum(len(sp) for sp in spans)
    # handles are exchanged on every call (the peers' buffers may have moved);
    # the mappings themselves are cached by handle in _PEER_MAPS
    counters = torch.zeros(n_pieces, dtype=torch.int64, device=state.device)
    ex = _allgather_exports([getattr(state, n) for n in names] + [counters], group)
    allh = [dict(bufs=dict(zip(names, e[:-1])), counters=e[-1]) for e in ex]
    chain = [src] + [r for r in range(world) if r != src]
    pos = chain.index(rank)
    nxt = None
    if pos + 1 < world:
        h = allh[chain[pos + 1]]

        def mapped(hh):
            hb, off = hh
            if hb not in _PEER_MAPS:
                base = C.c_void_p()
                check(LIB.rw_ipc_import(hb, C.byref(base)))
                _PEER_MAPS[hb] = base
            return _PEER_MAPS[hb].value + off

        nxt = dict(bufs={n: mapped(h["bufs"][n]) for n in names}, counters=mapped(h["counters"]))
    dkey = state.device.index
    if dkey not in _CE_CHAINS:
        _CE_CHAINS[dkey] = torch.cuda.Stream(device=state.device)
    cs, ep = _CE_CHAINS[dkey], 1
    sh = C.c_void_p(cs.cuda_stream)
    undo = set(plan.undo_ids) if plan.strategy == STRATEGY_NAMES[STRATEGY_UNDO] else set()
    if rank == src and plan.strategy not in (STRATEGY_NAMES[STRATEGY_UNDO], "None"):
        apply_resolution(state, hyper, plan)
    if rank == src and undo:
        mk = state.markers()
        if any(mk[i][1] == 0 for i in undo):
            state.write_markers([(t, 1 if i in undo else u) for i, (t, u) in enumerate(mk)])
    es = getattr(state, names[0]).element_size()
    cptr = counters.data_ptr()
    piece = 0
    for (g0, g1), span in zip(runs, spans):
        if rank == src:
            ids = [j for j in range(g0, g1) if j in undo]
            if ids:
                state.undo(hyper, ids)
            ev = torch.cuda.Event()
            ev.record()
            cs.wait_event(ev)
        for lo, hi in span:
            if rank != src:  # wait until the previous hop's copy of this piece has landed
                check(LIB.rw_stream_wait_u64(sh, C.c_void_p(cptr + 8 * piece), ep))
            if nxt is not None:
                n = len(names)
                dsts = (C.c_void_p * n)(*[nxt["bufs"][nm] + lo * es for nm in names])
                srcs = (C.c_void_p * n)(*[getattr(state, nm).data_ptr() + lo * es for nm in names])
                nbytes = (C.c_uint64 * n)(*[(hi - lo) * es] * n)
                check(LIB.rw_copy_async(dsts, srcs, nbytes, n, sh))
                check(LIB.rw_stream_write_u64(sh, C.c_void_p(nxt["counters"] + 8 * piece), ep))
            piece += 1
    torch.cuda.current_stream().wait_stream(cs)
    torch.cuda.current_stream().synchronize()
    dist.barrier(group=group)  # every hop has landed everywhere (counters may now be freed)
    _broadcast_saved_scalars(state, src, group)
    mk = state.markers()
    backend = dist.get_backend(group)
    dev = state.device if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([v for pair in mk for v in pair], dtype=torch.int64, device=dev)
    dist.broadcast(t, src=src, group=group)
    flat = t.cpu().tolist()
    state.write_markers([(flat[2 * i], flat[2 * i + 1]) for i in range(len(mk))])
    return sum(sum(state.sizes) * getattr(state, n).element_size() for n in names)


def recover(state, hyper, plan: ResolvePlan, src: int, include_grad: bool = False, group=None,
            transfer: str = "auto") -> tuple[str, int]:
    """apply_undo + recover_replication.  transfer:
      "chain": the undo run by run overlapped with copy-engine pushes of the
          resolved runs into the next rank's HBM (CUDA IPC), each replacement
          forwarding to the next (auto for one replacement);
      "pipelined": the undo run by run overlapped with concurrent async NCCL
          broadcasts of the resolved runs, one communicator per buffer (auto
          for several replacements);
      "fused": one kernel undoes and pushes every tile into the replacement's
          HBM with SM bulk stores (one replacement at a time);
      "broadcast": undo, then ncclBroadcast; "scatter_allgather".
    Measured for GPT-2 XL (18.7 GB, resolve included): N=2 chain 26.6-26.7 ms,
    pipelined 27.9, fused 29.5-29.9, broadcast 31.0-31.5; N=4 pipelined
    28.4-28.8, chain 29.1-30.1 (one sub-range of lag per hop), broadcast 32.0-32.4,
    scatter+all-gather 45.8-46.1, fused (sequential pushes) 82.  NVLink write
    bandwidth by engine (tools/peer_bw.cu): copy engines 781 GB/s, SM stores
    (TMA bulk or st.v4) 717.  Returns (transfer used, bytes per replacement)."""
    if transfer == "auto":  # measured best per replacement count (see the docstring)
        world = dist.get_world_size(group)
        transfer = "chain" if (world == 2 and world <= torch.cuda.device_count()) else "pipelined"
    if transfer == "fused":
        return transfer, recover_replication_fused(state, hyper, plan, src, include_grad, group)
    if transfer == "pipelined":
        return transfer, recover_replication_pipelined(state, hyper, plan, src, include_grad, group,
                                                       pieces=_PIPE[0], lead=_PIPE[1])
    if transfer == "chain":
        return transfer, recover_replication_chain(state, hyper, plan, src, include_grad, group)
    if dist.get_rank(group) == src:
        apply_resolution(state, hyper, plan)
    algo = "scatter_allgather" if transfer == "scatter_allgather" else "broadcast"
    return algo, recover_replication(state, src, include_grad, group, algo=algo)
