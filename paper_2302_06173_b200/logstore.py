"""Logging capture path and log files (logstore.cpp is absent).

Python mirror of the native logger in csrc/logger.cpp: ``Logger.log_send``
 enqueues a device tensor without blocking the producer stream
(GPU CRC32 + D2H on the logger's own stream, committed to "SWFT" chunk files
by a native thread); ``Logger.flush`` is flush_logs;
``load_log_dir`` fetches the records back for replay,
verifying every payload's CRC32 on the device (CorruptLog on mismatch) and
returning a ``replay.BoundaryLog`` keyed by (iteration, micro-batch).
"""
from __future__ import annotations

import collections
import ctypes as C
import glob
import os
from typing import Iterable, Iterator

import torch

from ._lib import LIB, RwError, check

RW_LOG_ACTIVATION, RW_LOG_GRADIENT = 0, 1
_DT = {torch.float32: 0, torch.float64: 1, torch.bfloat16: 2}
_DT_INV = {v: k for k, v in _DT.items()}


class rw_log_record(C.Structure):
    _fields_ = [("sender", C.c_uint32), ("receiver", C.c_uint32), ("iteration", C.c_uint64),
                ("mb", C.c_uint32), ("direction", C.c_uint32), ("dtype", C.c_uint32), ("ndim", C.c_uint32),
                ("shape", C.c_uint64 * 4), ("payload_bytes", C.c_uint64), ("crc32", C.c_uint32),
                ("_pad", C.c_uint32)]


_vp, _u32, _u64 = C.c_void_p, C.c_uint32, C.c_uint64
for _n, (_r, _a) in {
    "rw_crc32_device": (C.c_int, [_vp, _u64, _vp, _vp]),
    "rw_logger_create": (C.c_int, [C.POINTER(_vp), C.c_char_p, _u32, _u32, _u64, C.c_int32]),
    "rw_logger_log": (C.c_int, [_vp, C.POINTER(rw_log_record), _vp, _vp]),
    "rw_logger_flush": (C.c_int, [_vp, C.POINTER(_u64)]),
    "rw_logger_destroy": (C.c_int, [_vp]),
    "rw_logger_stream": (_vp, [_vp]),
    "rw_log_open": (C.c_int, [C.POINTER(_vp), C.c_char_p, C.POINTER(_u32)]),
    "rw_log_next": (C.c_int, [_vp, C.POINTER(rw_log_record), _vp, _u64, C.POINTER(C.c_int32)]),
    "rw_log_close": (None, [_vp]),
}.items():
    _f = getattr(LIB, _n)
    _f.restype, _f.argtypes = _r, _a


def _stream(stream=None) -> _vp:
    return _vp((stream or torch.cuda.current_stream()).cuda_stream)


def crc32_device(t: torch.Tensor, stream=None) -> int:
    """CRC32 (wire.cpp:31-38) of a contiguous device tensor's bytes, on the GPU."""
    t = t.contiguous()
    out = torch.zeros(1, dtype=torch.int32, device=t.device)
    check(LIB.rw_crc32_device(_vp(t.data_ptr()), t.numel() * t.element_size(), _vp(out.data_ptr()),
                              _stream(stream)))
    return int(out.item()) & 0xFFFFFFFF


class Logger:
    """Upstream-backup logger of one machine.  pinned_bytes is
    the host staging slab: a few boundary records (a config-4 record is 134 MB)
    so log_send rarely waits for the writer lanes."""

    def __init__(self, directory: str, machine: int, chunk_records: int = 64,
                 pinned_bytes: int = 1 << 30, device: int | None = None):
        os.makedirs(directory, exist_ok=True)
        self.dir = directory
        self._h = _vp()
        dev = torch.cuda.current_device() if device is None else device
        check(LIB.rw_logger_create(C.byref(self._h), directory.encode(), machine, chunk_records, pinned_bytes,
                                   dev))
        # payloads in flight: (event on the logger's copy stream after the
        # record's D2H, tensor).  Trimmed on every log_send as the copies
        # complete, so device memory is held only while the D2H still reads it.
        self._copy_stream = torch.cuda.ExternalStream(LIB.rw_logger_stream(self._h), device=dev)
        self._inflight: collections.deque = collections.deque()

    def log_send(self, t: torch.Tensor, sender: int, receiver: int, iteration: int, mb: int, direction: int,
                 stream=None) -> None:
        """Enqueue the message tensor `t` (device).  The producer stream is not
        blocked; `t` must stay unmodified until the copy has been issued on the
        logger stream (it is ordered after the current work on `stream`)."""
        t = t.contiguous()
        r = rw_log_record()
        r.sender, r.receiver, r.iteration, r.mb, r.direction = sender, receiver, iteration, mb, direction
        r.dtype = _DT[t.dtype]
        r.ndim = t.dim()
        for i, s in enumerate(t.shape):
            r.shape[i] = s
        r.payload_bytes = t.numel() * t.element_size()
        check(LIB.rw_logger_log(self._h, C.byref(r), _vp(t.data_ptr()), _stream(stream)))
        ev = torch.cuda.Event()
        ev.record(self._copy_stream)  # after this record's CRC + D2H on the logger stream
        self._inflight.append((ev, t))
        while self._inflight and self._inflight[0][0].query():
            self._inflight.popleft()

    def flush(self) -> int:
        n = _u64()
        check(LIB.rw_logger_flush(self._h, C.byref(n)))
        self._inflight.clear()  # flush waited for every copy
        return n.value

    def close(self) -> None:
        if self._h.value:
            st = LIB.rw_logger_destroy(self._h)
            self._h = _vp()
            self._inflight.clear()
            check(st)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_chunk(path: str, max_payload: int = 1 << 30) -> Iterator[tuple[rw_log_record, torch.Tensor]]:
    """Yield (record, pinned host payload bytes) from one chunk file."""
    h = _vp()
    m = _u32()
    check(LIB.rw_log_open(C.byref(h), path.encode(), C.byref(m)))
    try:
        # pinned when a device is present (fast H2D for replay); the reader itself is host code
        cap = max(1, min(max_payload, os.path.getsize(path)))  # a record never exceeds its file
        buf = torch.empty(cap, dtype=torch.uint8, pin_memory=torch.cuda.is_available())
        while True:
            r = rw_log_record()
            eof = C.c_int32()
            check(LIB.rw_log_next(h, C.byref(r), _vp(buf.data_ptr()), buf.numel(), C.byref(eof)))
            if eof.value:
                return
            yield r, buf[:r.payload_bytes].clone()
    finally:
        LIB.rw_log_close(h)


def load_log_dir(directory: str, device=None, max_payload: int = 1 << 30, machine: int | None = None,
                 receivers: Iterable[int] | None = None, min_iteration: int = 0):
    """fetch_logs for replay: every committed chunk file of the
    directory (optionally one sender machine's), keeping the records addressed
    to `receivers` (the failed group's first and last stage: its inbound
    activations and gradients; default all) from iteration `min_iteration` on,
    payloads moved to the device and CRC-verified there.  Returns a
    replay.BoundaryLog."""
    from .replay import BoundaryLog
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    pat = "m*.swft" if machine is None else f"m{machine:04d}_*.swft"
    log = BoundaryLog()
    recv = None if receivers is None else set(int(x) for x in receivers)
    for path in sorted(glob.glob(os.path.join(directory, pat))):
        for r, payload in read_chunk(path, max_payload):
            if (recv is not None and int(r.receiver) not in recv) or int(r.iteration) < min_iteration:
                continue
            d = payload.to(dev, non_blocking=True)
            if crc32_device(d) != r.crc32:
                raise RwError(15, f"CorruptLog: CRC mismatch in {path} (it {r.iteration}, mb {r.mb})")
            shape = [int(r.shape[i]) for i in range(r.ndim)]
            t = d.view(_DT_INV[r.dtype]).view(shape)
            key = (int(r.iteration), int(r.mb))
            (log.acts if r.direction == RW_LOG_ACTIVATION else log.grads)[key] = t
    return log
