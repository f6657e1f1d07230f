"""Global checkpoint store feeding replay (SPEC:389-392 CheckpointManifest,
SPEC:423-438 write_checkpoint / load_checkpoint / gc_logs; no reference
source — SURVEY §8f rank 3).

The byte mover is native (csrc/checkpoint.cpp): device buffers stream
through a pinned ring (D2H overlapped with write(2); pread overlapped with
H2D), CRC32 on the GPU, fsync'd blobs, per-worker manifests and one global
``MANIFEST_<iteration>`` published by rename — the checkpoint is visible iff
every blob of every worker is durable.

A worker's checkpoint holds, per DeviceState (prefix ``s<k>.``): x, m, v
(vmax for AMSGrad, g when asked) plus a JSON meta blob with the layout, the
update-progress markers and LAMB's saved trust ratios ("per-worker state
blob references (params, optimizer state, step counters, RNG positions)",
SPEC:390).  ``extra`` carries caller state such as RNG positions.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Sequence

import torch
import torch.distributed as dist

from ._lib import LAMB, LIB, RwError, check


class rw_blob(C.Structure):
    _fields_ = [("name", C.c_char_p), ("data", C.c_void_p), ("bytes", C.c_uint64), ("on_host", C.c_uint32),
                ("pad", C.c_uint32)]


_vp, _u32, _u64 = C.c_void_p, C.c_uint32, C.c_uint64
for _n, (_r, _a) in {
    "rw_ckpt_write": (C.c_int, [C.c_char_p, _u64, _u32, C.POINTER(rw_blob), _u32, _u32, _vp]),
    "rw_ckpt_commit": (C.c_int, [C.c_char_p, _u64, _u32]),
    "rw_ckpt_latest": (C.c_int, [C.c_char_p, C.POINTER(_u64)]),
    "rw_ckpt_blob_bytes": (C.c_int, [C.c_char_p, _u64, _u32, C.c_char_p, C.POINTER(_u64)]),
    "rw_ckpt_load": (C.c_int, [C.c_char_p, _u64, _u32, C.POINTER(rw_blob), _u32, _vp]),
    "rw_log_gc": (C.c_int, [C.c_char_p, C.c_char_p, _u64, C.POINTER(_u32)]),
}.items():
    _f = getattr(LIB, _n)
    _f.restype, _f.argtypes = _r, _a

NO_CRASH = 0xFFFFFFFF


def _stream(stream=None):
    if stream is None and torch.cuda.is_available():
        stream = torch.cuda.current_stream()
    return _vp(stream.cuda_stream if stream is not None else None)


def _bufs(state, include_grad: bool):
    names = ["x"] + (["g"] if include_grad else []) + [n for n in ("m", "v", "vmax")
                                                       if getattr(state, n) is not None]
    return [(n, getattr(state, n)) for n in names]


def _meta(states: Sequence, include_grad: bool, extra: dict | None) -> bytes:
    per = []
    for st in states:
        per.append(dict(sizes=st.sizes, offsets=st.offsets, total=st.total, kind=st.kind,
                        dtype=str(st.dtype), markers=st.markers(),
                        saved_scalars=[st.saved_scalars(i) for i in range(st.num_groups)]
                        if getattr(st, "kind", None) == LAMB else None,
                        buffers=[n for n, _ in _bufs(st, include_grad)]))
    return json.dumps(dict(version=1, states=per, extra=extra or {}), sort_keys=True).encode()


def write_checkpoint(states, ckpt_dir: str, iteration: int, worker: int | None = None, group=None,
                     include_grad: bool = False, extra: dict | None = None,
                     crash_after_blobs: int | None = None, commit: bool = True, stream=None) -> None:
    """write_checkpoint for this worker's states; with a process
    group every rank writes its own blobs, then rank 0 publishes the manifest
    after a barrier (all workers at the same iteration boundary)."""
    states = list(states) if isinstance(states, (list, tuple)) else [states]
    distributed = dist.is_available() and dist.is_initialized()
    if worker is None:
        worker = dist.get_rank(group) if distributed else 0
    meta = _meta(states, include_grad, extra)
    keep = [C.create_string_buffer(meta, len(meta))]
    blobs = []
    for k, st in enumerate(states):
        for n, t in _bufs(st, include_grad):
            blobs.append(rw_blob(f"s{k}.{n}".encode(), _vp(t.data_ptr()), t.numel() * t.element_size(), 0, 0))
    blobs.append(rw_blob(b"meta.json", C.cast(keep[0], _vp), len(meta), 1, 0))
    arr = (rw_blob * len(blobs))(*blobs)
    crash = NO_CRASH if crash_after_blobs is None else int(crash_after_blobs)
    check(LIB.rw_ckpt_write(ckpt_dir.encode(), iteration, worker, arr, len(blobs), crash, _stream(stream)))
    if not commit:
        return
    if distributed:
        dist.barrier(group=group)
        if dist.get_rank(group) == 0:
            check(LIB.rw_ckpt_commit(ckpt_dir.encode(), iteration, dist.get_world_size(group)))
        dist.barrier(group=group)
    else:
        check(LIB.rw_ckpt_commit(ckpt_dir.encode(), iteration, 1))


def commit_checkpoint(ckpt_dir: str, iteration: int, workers: int) -> None:
    """Publish MANIFEST_<iteration> once every one of `workers` workers has
    written its blobs (write_checkpoint(..., commit=False) per worker): the
    global checkpoint becomes visible atomically."""
    check(LIB.rw_ckpt_commit(ckpt_dir.encode(), iteration, workers))


def latest_checkpoint(ckpt_dir: str) -> int:
    """Highest committed iteration (NoCheckpoint if none)."""
    it = C.c_uint64()
    check(LIB.rw_ckpt_latest(ckpt_dir.encode(), C.byref(it)))
    return it.value


def load_checkpoint(states, ckpt_dir: str, iteration: int | None = None, worker: int | None = None,
                    group=None, stream=None) -> tuple[int, dict]:
    """load_checkpoint: restore x, m, v (g, vmax when saved),
    the markers and LAMB's saved ratios of each state, bit for bit.  Returns
    (iteration, extra)."""
    states = list(states) if isinstance(states, (list, tuple)) else [states]
    if worker is None:
        worker = dist.get_rank(group) if (dist.is_available() and dist.is_initialized()) else 0
    if iteration is None:
        iteration = latest_checkpoint(ckpt_dir)
    nb = C.c_uint64()
    check(LIB.rw_ckpt_blob_bytes(ckpt_dir.encode(), iteration, worker, b"meta.json", C.byref(nb)))
    mbuf = C.create_string_buffer(nb.value)
    one = (rw_blob * 1)(rw_blob(b"meta.json", C.cast(mbuf, _vp), nb.value, 1, 0))
    check(LIB.rw_ckpt_load(ckpt_dir.encode(), iteration, worker, one, 1, _stream(stream)))
    meta = json.loads(mbuf.raw[:nb.value].decode())
    if len(meta["states"]) != len(states):
        raise RwError(2, "ShapeMismatch: checkpoint holds %d states, %d given" % (len(meta["states"]), len(states)))
    blobs = []
    for k, (st, m) in enumerate(zip(states, meta["states"])):
        if m["sizes"] != st.sizes or m["dtype"] != str(st.dtype) or m["kind"] != st.kind:
            raise RwError(2, f"ShapeMismatch: state {k} layout/dtype/kind differs from the checkpoint")
        for n in m["buffers"]:
            t = getattr(st, n)
            if t is None:
                raise RwError(2, f"ShapeMismatch: state {k} has no buffer {n}")
            blobs.append(rw_blob(f"s{k}.{n}".encode(), _vp(t.data_ptr()), t.numel() * t.element_size(), 0, 0))
    arr = (rw_blob * max(len(blobs), 1))(*blobs)
    check(LIB.rw_ckpt_load(ckpt_dir.encode(), iteration, worker, arr, len(blobs), _stream(stream)))
    for st, m in zip(states, meta["states"]):
        st.write_markers([tuple(x) for x in m["markers"]], stream)
        if m["saved_scalars"] is not None:
            for i, vals in enumerate(m["saved_scalars"]):
                st.set_saved_scalars(i, vals, stream)
    return iteration, meta["extra"]


def gc_logs(log_dir: str, ckpt_dir: str, ckpt_iteration: int) -> int:
    """gc_logs: delete log chunks wholly before the committed
    checkpoint; returns the number of chunk files removed (idempotent)."""
    n = C.c_uint32()
    check(LIB.rw_log_gc(log_dir.encode(), ckpt_dir.encode(), ckpt_iteration, C.byref(n)))
    return n.value


def stored_bytes(directory: str) -> int:
    """Bytes under a directory (log-volume accounting for the GC bound)."""
    tot = 0
    for root, _, files in os.walk(directory):
        for f in files:
            tot += os.path.getsize(os.path.join(root, f))
    return tot
