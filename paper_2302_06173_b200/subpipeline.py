"""Stage-per-GPU sub-pipeline replay (replay way (i)).

The failed group's stages are folded onto the d GPUs in contiguous blocks
(worker w holds stages [w*p/d, (w+1)*p/d)); micro-batches flow through the
workers in the 1F1B order of schedule.cpp (warm-up forwards, one-forward-
one-backward, cool-down backwards), activations forward and gradients back
across the worker boundaries.  Each worker steps its own stages after the
iteration, so no gradient merge is needed; the price is the pipeline bubble
(d-1)/(m+d-1) that parallel recovery (replay.recover_parallel, way (ii))
avoids.

Boundary tensors move like the copy-engine merge (merge.py): cudaMemcpyAsync
into the neighbour's CUDA-IPC-mapped receive slot (one per micro-batch), then
an epoch counter written from the same copy stream (cuStreamWriteValue64);
the neighbour's compute stream waits on it (cuStreamWaitValue64) -- no SM is
taken from the persistent GEMM grids.  The math is replay_group's, so the
result is bit-identical to the sequential replay of the whole group.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import torch
import torch.distributed as dist

from ._lib import LIB, RwError, check
from .replay import BoundaryLog, Stage, mse_grad, synth_inputs, synth_targets


def one_f_one_b(workers: int, m: int, w: int) -> list[tuple[str, int]]:
    """The 1F1B order of worker w (schedule.cpp:25-84 restated for one
    worker): min(d-1-w, m) warm-up forwards, then alternate F/B, then the
    remaining backwards; backwards run in ascending micro-batch order."""
    warm = min(workers - 1 - w, m)
    ops, f, b = [], 0, 0
    for _ in range(warm):
        ops.append(("F", f))
        f += 1
    while f < m:
        ops.append(("F", f))
        f += 1
        ops.append(("B", b))
        b += 1
    while b < m:
        ops.append(("B", b))
        b += 1
    return ops


def split_stages(p: int, d: int, w: int) -> range:
    """Contiguous block of stages of worker w."""
    return range(p * w // d, p * (w + 1) // d)


class SubPipeline:
    """Worker `rank` of a d-worker sub-pipeline over `stages` (this worker's
    contiguous block, in order)."""

    def __init__(self, stages: Sequence[Stage], m: int, rows: int, dim: int, group=None):
        from .recovery import _PEER_MAPS, _export
        self.stages = list(stages)
        if not self.stages:
            raise RwError(18, "InvalidConfig: every sub-pipeline worker needs at least one stage (p >= d)")
        self.m, self.rows, self.dim, self.group = m, rows, dim, group
        self.d, self.w = dist.get_world_size(group), dist.get_rank(group)
        self.dev = self.stages[0].device
        bf = torch.bfloat16
        # receive slots: activations from w-1, gradients from w+1 (one per micro-batch)
        self.act_in = [torch.empty(rows, dim, dtype=bf, device=self.dev) for _ in range(m)] if self.w > 0 else []
        self.grad_in = ([torch.empty(rows, dim, dtype=bf, device=self.dev) for _ in range(m)]
                        if self.w < self.d - 1 else [])
        self.counters = torch.zeros(2, m, dtype=torch.int64, device=self.dev)  # [0]: act, [1]: grad
        self.epoch = 0
        self.copy_stream = torch.cuda.Stream(device=self.dev)
        # the compute runs on its own stream: a value-wait on the legacy default
        # stream would also hold back the copy stream that feeds the neighbour
        self.stream = torch.cuda.Stream(device=self.dev)
        mine = dict(act=[_export(t) for t in self.act_in], grad=[_export(t) for t in self.grad_in],
                    counters=_export(self.counters))
        allh: list = [None] * self.d
        dist.all_gather_object(allh, mine, group=group)

        def mapped(h):
            hb, off = h
            if hb not in _PEER_MAPS:
                base = C.c_void_p()
                check(LIB.rw_ipc_import(hb, C.byref(base)))
                _PEER_MAPS[hb] = base
            return _PEER_MAPS[hb].value + off

        self.next = None if self.w == self.d - 1 else dict(
            act=[mapped(x) for x in allh[self.w + 1]["act"]], counters=mapped(allh[self.w + 1]["counters"]))
        self.prev = None if self.w == 0 else dict(
            grad=[mapped(x) for x in allh[self.w - 1]["grad"]], counters=mapped(allh[self.w - 1]["counters"]))

    # ---- boundary transfers ----
    def _send(self, t: torch.Tensor, dst: int, counter: int) -> None:
        ev = torch.cuda.Event()
        ev.record()
        self.copy_stream.wait_event(ev)
        sh = C.c_void_p(self.copy_stream.cuda_stream)
        n = t.numel() * t.element_size()
        check(LIB.rw_copy_async((C.c_void_p * 1)(dst), (C.c_void_p * 1)(t.data_ptr()), (C.c_uint64 * 1)(n), 1, sh))
        check(LIB.rw_stream_write_u64(sh, C.c_void_p(counter), self.epoch))
        t.record_stream(self.copy_stream)

    def _wait(self, kind: int, mb: int) -> None:
        addr = self.counters.data_ptr() + (kind * self.m + mb) * 8
        check(LIB.rw_stream_wait_u64(C.c_void_p(torch.cuda.current_stream().cuda_stream), C.c_void_p(addr),
                                     self.epoch))

    # ---- one replayed iteration ----
    def iteration(self, log: BoundaryLog, it: int, seed: int, hyper, first: bool, last: bool) -> None:
        caller = torch.cuda.current_stream()
        self.stream.wait_stream(caller)
        with torch.cuda.stream(self.stream):
            self._iteration(log, it, seed, hyper, first, last)
        caller.wait_stream(self.stream)

    def _iteration(self, log: BoundaryLog, it: int, seed: int, hyper, first: bool, last: bool) -> None:
        self.epoch += 1
        rows, dim, dev = self.rows, self.dim, self.dev
        cache = {}
        for op, mb in one_f_one_b(self.d, self.m, self.w):
            if op == "F":
                if self.w > 0:
                    self._wait(0, mb)
                    x = self.act_in[mb]
                elif first:
                    x = synth_inputs(seed, it, mb, rows, dim, device=dev)
                else:
                    x = log.get("act", it, mb, dev)
                    if x is None:
                        raise RwError(14, f"MissingLogData: activation ({it}, {mb})")
                all_acts = []
                for st in self.stages:
                    acts = st.new_acts(rows, x)
                    x = st.forward(acts)
                    all_acts.append(acts)
                cache[mb] = all_acts
                if self.next is not None:
                    self._send(x, self.next["act"][mb], self.next["counters"] + (0 * self.m + mb) * 8)
            else:
                all_acts = cache.pop(mb)
                if self.w < self.d - 1:
                    self._wait(1, mb)
                    g = self.grad_in[mb]
                elif last:
                    g = mse_grad(all_acts[-1][-1], synth_targets(seed, it, mb, rows, dim, device=dev), self.m)
                else:
                    g = log.get("grad", it, mb, dev)
                    if g is None:
                        raise RwError(14, f"MissingLogData: gradient ({it}, {mb})")
                n = len(self.stages)
                for k in range(n - 1, -1, -1):
                    # boundary to the previous worker: plain dgrad (sent as bf16, like
                    # the original run); inside the worker: fused with the dtanh
                    need_out = k > 0 or self.w > 0
                    gout = torch.empty(rows, self.stages[k].dims[0], dtype=torch.bfloat16,
                                       device=dev) if need_out else None
                    self.stages[k].backward(all_acts[k], g, gout, accumulate=mb > 0, grad_in_is_dz=k < n - 1,
                                            prev_y=all_acts[k - 1][-1] if k > 0 else None)
                    g = gout
                if self.prev is not None:
                    self._send(g, self.prev["grad"][mb], self.prev["counters"] + (1 * self.m + mb) * 8)
        for st in reversed(self.stages):
            st.step(hyper)


def recover_subpipeline(pipe: SubPipeline, log: BoundaryLog, it0: int, it1: int, seed: int, hyper,
                        first: bool, last: bool) -> int:
    """recover_replay of the group over [it0, it1) on the sub-pipeline."""
    for it in range(it0, it1):
        pipe.iteration(log, it, seed, hyper, first, last)
    return it1 - it0
