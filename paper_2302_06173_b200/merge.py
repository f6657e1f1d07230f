"""Parallel-recovery merge over the copy engines.

The helpers of recover_parallel hold per-micro-batch fp32 gradients of every
stage; the merged gradient is the left-to-right sum over micro-batches
0..m-1 (ordered_sum, bit-identical to the sequential replay).  The flat
gradient of a stage is sharded over the d ranks; rank j owns shard j.

Data movement here uses no SM at all, so it overlaps the replay GEMMs without
stalling their persistent grids (an NCCL-kernel overlap does stall them):

  scatter  as soon as a stage's gradients of this helper's micro-batches are
           complete, shard j of each is copied (cudaMemcpyAsync, DMA over
           NVLink) into rank j's receive arena slot for that micro-batch, then
           the epoch is written into rank j's counter for (stage, sender) from
           the same copy stream;
  reduce   rank j's merge stream waits (cuStreamWaitValue64) for every
           sender's counter, then sums the m shards in ascending micro-batch
           order into its slice of the full gradient buffer;
  gather   the merged shard is copied into every peer's full-gradient buffer
           + a second counter; each rank waits for all of them and steps.

Receive arenas, full-gradient buffers and counters are allocated once,
exported with CUDA IPC and mapped by every peer (one all_gather_object).
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import torch
import torch.distributed as dist

from ._lib import LIB, check
from .optim import ordered_sum


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class CopyEngineMerger:
    def __init__(self, numels: Sequence[int], m: int, group=None):
        self.d, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.m, self.group = m, group
        self.dev = torch.device("cuda", torch.cuda.current_device())
        d = self.d
        self.P = list(numels)
        self.chunk = [((p + d - 1) // d + 63) // 64 * 64 for p in self.P]
        L = len(self.P)
        # arena[k]: [m, chunk_k] receive slots (by micro-batch); full[k]: [d * chunk_k]
        self.arena = [torch.empty(m * c, dtype=torch.float32, device=self.dev) for c in self.chunk]
        self.full = [torch.zeros(d * c, dtype=torch.float32, device=self.dev) for c in self.chunk]
        # counters[phase, k, sender]: epochs written by peers (0 = never)
        self.counters = torch.zeros(2, L, d, dtype=torch.int64, device=self.dev)
        self.epoch = 0
        self.copy_stream = torch.cuda.Stream(device=self.dev)
        self.merge_stream = torch.cuda.Stream(device=self.dev)
        from .recovery import _PEER_MAPS, _export
        mine = dict(arena=[_export(a) for a in self.arena], full=[_export(f) for f in self.full],
                    counters=_export(self.counters))
        allh: list = [None] * d
        dist.all_gather_object(allh, mine, group=group)

        def mapped(h):
            hb, off = h
            if hb not in _PEER_MAPS:
                base = C.c_void_p()
                check(LIB.rw_ipc_import(hb, C.byref(base)))
                _PEER_MAPS[hb] = base
            return _PEER_MAPS[hb].value + off

        self.peer = {}
        for r in range(d):
            if r == self.rank:
                continue
            h = allh[r]
            self.peer[r] = dict(arena=[mapped(x) for x in h["arena"]], full=[mapped(x) for x in h["full"]],
                                counters=mapped(h["counters"]))

    def bounds(self, k: int, j: int) -> tuple[int, int]:
        c, P = self.chunk[k], self.P[k]
        return min(P, j * c), min(P, (j + 1) * c)

    def _counter_addr(self, r: int, phase: int, k: int, sender: int) -> int:
        L = len(self.P)
        base = self.peer[r]["counters"] if r != self.rank else _ptr(self.counters)
        return base + ((phase * L + k) * self.d + sender) * 8

    def begin_iteration(self) -> None:
        self.epoch += 1

    def scatter(self, k: int, bufs: dict) -> None:
        """Stage k's gradients of this helper's micro-batches are complete on
        the current stream: ship shard j of each to rank j (DMA)."""
        ev = torch.cuda.Event()
        ev.record()
        self.copy_stream.wait_event(ev)
        dsts, srcs, nbytes = [], [], []
        for mb, buf in sorted(bufs.items()):
            for j in range(self.d):
                if j == self.rank:
                    continue
                lo, hi = self.bounds(k, j)
                if hi <= lo:
                    continue
                dsts.append(self.peer[j]["arena"][k] + mb * self.chunk[k] * 4)
                srcs.append(_ptr(buf) + lo * 4)
                nbytes.append((hi - lo) * 4)
        sh = C.c_void_p(self.copy_stream.cuda_stream)
        n = len(dsts)
        if n:
            check(LIB.rw_copy_async((C.c_void_p * n)(*dsts), (C.c_void_p * n)(*srcs), (C.c_uint64 * n)(*nbytes),
                                    n, sh))
        for j in range(self.d):  # also to ranks that got nothing from us: they wait on every sender
            if j != self.rank:
                check(LIB.rw_stream_write_u64(sh, C.c_void_p(self._counter_addr(j, 0, k, self.rank)), self.epoch))
        for b in bufs.values():
            b.record_stream(self.copy_stream)

    def reduce_gather(self, k: int, own: dict, wait: bool = True):
        """Ordered sum of this rank's shard of stage k (own micro-batches from
        `own`, the others from the arena), then the gather, all on the merge
        stream.  wait=True: the current stream waits and the full merged
        gradient is returned; wait=False: returns (gradient, event) so the
        caller can keep computing and wait on the event before the step."""
        d, rank = self.d, self.rank
        ms = self.merge_stream
        sh = C.c_void_p(ms.cuda_stream)
        ev = torch.cuda.Event()
        ev.record()
        ms.wait_event(ev)
        for s in range(d):
            if s != rank:
                check(LIB.rw_stream_wait_u64(sh, C.c_void_p(self._counter_addr(rank, 0, k, s)), self.epoch))
        lo, hi = self.bounds(k, rank)
        c = self.chunk[k]
        with torch.cuda.stream(ms):
            if hi > lo:
                parts = [own[mb][lo:hi] if mb in own else self.arena[k][mb * c:mb * c + (hi - lo)]
                         for mb in range(self.m)]
                ordered_sum(parts, out=self.full[k][rank * c:rank * c + (hi - lo)], stream=ms)
        # gather: our merged shard into every peer's full buffer, then the epoch
        dsts, srcs, nbytes = [], [], []
        for j in range(d):
            if j != rank and hi > lo:
                dsts.append(self.peer[j]["full"][k] + rank * c * 4)
                srcs.append(_ptr(self.full[k]) + rank * c * 4)
                nbytes.append((hi - lo) * 4)
        n = len(dsts)
        if n:
            check(LIB.rw_copy_async((C.c_void_p * n)(*dsts), (C.c_void_p * n)(*srcs), (C.c_uint64 * n)(*nbytes),
                                    n, sh))
        for j in range(d):
            if j != rank:
                check(LIB.rw_stream_write_u64(sh, C.c_void_p(self._counter_addr(j, 1, k, rank)), self.epoch))
        for s in range(d):
            if s != rank:
                check(LIB.rw_stream_wait_u64(sh, C.c_void_p(self._counter_addr(rank, 1, k, s)), self.epoch))
        done = torch.cuda.Event()
        done.record(ms)
        for b in own.values():
            b.record_stream(ms)
        if not wait:
            return self.full[k][:self.P[k]], done
        torch.cuda.current_stream().wait_event(done)
        return self.full[k][:self.P[k]]
