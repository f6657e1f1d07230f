"""The copy-engine transfer primitives of replica recovery and the parallel
merge (rw_copy_async, rw_stream_write_u64 / rw_stream_wait_u64), on ONE GPU:
the same stream-ordered epoch protocol the chain transfer runs between
devices (recovery.recover_replication_chain: the survivor copies resolved runs
and bumps the receiver's counter; the receiver's stream waits on it), here
between two streams of one device, so a single-GPU box exercises it too.

* the consumer stream never reads a run before its epoch was written (its
  checksum of every run equals the source's, although the producer is held
  back by a spin before each run);
* runs land bit for bit; a batch of copies in one call moves every run;
* the undo of a resolved run pipelined with its copy (the chain's pattern)
  yields the locally undone state in the receiver's buffers.
"""
import ctypes as C

import pytest
import torch

from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper, seeded_fill_
from paper_2302_06173_b200._lib import LIB, check

pytestmark = pytest.mark.gpu


def _vp(x):
    return C.c_void_p(x)


def test_epoch_ordered_copy_between_streams():
    n_runs, run = 8, 1 << 20
    src = torch.empty(n_runs * run, dtype=torch.float32, device="cuda")
    seeded_fill_(src, 99)
    dst = torch.zeros_like(src)
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    sums = torch.zeros(n_runs, dtype=torch.float64, device="cuda")
    prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
    # The producer is enqueued first: on ONE device two streams may share a
    # hardware queue, and a value-wait queued ahead of the work it waits for
    # would then block that work (across devices, as in the chain, it cannot).
    for k in range(n_runs):  # producer, deliberately slow: spin, copy run k, publish epoch k+1
        with torch.cuda.stream(prod):
            torch.cuda._sleep(200_000)
        d = (C.c_void_p * 1)(dst.data_ptr() + 4 * k * run)
        s = (C.c_void_p * 1)(src.data_ptr() + 4 * k * run)
        nb = (C.c_uint64 * 1)(4 * run)
        check(LIB.rw_copy_async(d, s, nb, 1, _vp(prod.cuda_stream)))
        check(LIB.rw_stream_write_u64(_vp(prod.cuda_stream), _vp(counter.data_ptr()), k + 1))
    for k in range(n_runs):  # consumer: wait for epoch k+1, then read run k
        check(LIB.rw_stream_wait_u64(_vp(cons.cuda_stream), _vp(counter.data_ptr()), k + 1))
        with torch.cuda.stream(cons):
            sums[k] = dst[k * run:(k + 1) * run].double().sum()
    torch.cuda.synchronize()
    assert torch.equal(dst, src)
    ref = torch.stack([src[k * run:(k + 1) * run].double().sum() for k in range(n_runs)])
    assert torch.equal(sums, ref)  # every run was read only after it landed
    assert int(counter.item()) == n_runs


def test_batched_copies_and_pipelined_undo_push():
    """The chain pattern on one device: resolved runs of an Adam state are
    undone in place and each run's x, m, v is copied (one batched call) into a
    second state as soon as its undo is done; the receiver equals a plain
    local undo bit for bit."""
    sizes = [3000, 77, 5000, 64, 12345, 999, 4096, 2]
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    a, ref = DeviceState(sizes, kind=ADAM), DeviceState(sizes, kind=ADAM)
    for st in (a, ref):
        for i, t in enumerate((st.x, st.g, st.m, st.v)):
            seeded_fill_(t, 10 + i)
        st.v.abs_()
        st.write_markers([(5, 0)] * len(sizes))
        st.step(h)
    ref.undo(h)
    b = DeviceState(sizes, kind=ADAM)
    runs = [[7, 6, 5], [4, 3], [2, 1, 0]]  # reverse update order, contiguous runs of groups
    stream = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    for ids in runs:
        a.undo(h, ids)
        ev = torch.cuda.Event()
        ev.record(stream)
        copy.wait_event(ev)
        lo = min(a.offsets[i] for i in ids)
        hi = max(a.offsets[i] + a.sizes[i] for i in ids)
        names = ("x", "m", "v")
        d = (C.c_void_p * 3)(*[getattr(b, k).data_ptr() + 4 * lo for k in names])
        s = (C.c_void_p * 3)(*[getattr(a, k).data_ptr() + 4 * lo for k in names])
        nb = (C.c_uint64 * 3)(*[4 * (hi - lo)] * 3)
        check(LIB.rw_copy_async(d, s, nb, 3, _vp(copy.cuda_stream)))
    torch.cuda.synchronize()
    for k in ("x", "m", "v"):
        for o, n in zip(ref.offsets, ref.sizes):
            assert torch.equal(getattr(b, k)[o:o + n], getattr(ref, k)[o:o + n]), k
