"""Host-side mirror of the reference optimizer API over the B200 kernels.

Reference: /root/reference/proj/core/include/rewind/optim.hpp and
src/optim.cpp.  ``OptimizerHyper`` mirrors optim.hpp:34-50, ``ParamBlock``
fields become one *group* of a flat device state (x, g, m, v as separate HBM
arrays, 256-byte aligned groups), and ``optimizer_step`` /
``optimizer_undo`` keep the reference names, argument meaning and error
behaviour (``RwError`` carries the same ``Err`` code ``rewind::Error`` would).

torch is used only to own device memory and streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import torch

from . import _lib
from ._lib import (ADAM, ADAMW, AMSGRAD, F32, F64, LAMB, LIB, SGD, SGDM, RwError, check,
                   rw_group, rw_hyper)

ALIGN_ELEMS = 64  # 256 B for fp32: 128-bit vector access never straddles groups

_KIND_NAMES = {"sgd": SGD, "sgdm": SGDM, "sgd_momentum": SGDM, "adam": ADAM, "adamw": ADAMW,
               "lamb": LAMB, "amsgrad": AMSGRAD}


TRUST_DEPTH = 8  # RW_LAMB_TRUST_DEPTH (include/rewind_b200.h)


def optimizer_from_name(name: str) -> int | None:
    """optimizer_from_name, optim.cpp:25-33."""
    return _KIND_NAMES.get(name)


def invertibility_check(kind: int) -> int:
    """invertibility_check, optim.hpp:32 / optim.cpp:35-48."""
    return LIB.rw_invertibility_check(kind)


@dataclass
class OptimizerHyper:
    """OptimizerHyper, optim.hpp:34-50 (same fields and defaults)."""

    kind: int = SGD
    lr: float = 0.01
    lr_table: list[tuple[int, float]] = field(default_factory=list)
    weight_decay: float = 0.0
    momentum: float = 0.9
    dampening: float = 0.0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    require_invertible: bool = False

    def to_c(self) -> rw_hyper:
        h = rw_hyper()
        h.kind = self.kind
        h.require_invertible = 1 if self.require_invertible else 0
        h.lr = self.lr
        h.weight_decay = self.weight_decay
        h.momentum = self.momentum
        h.dampening = self.dampening
        h.beta1 = self.beta1
        h.beta2 = self.beta2
        h.eps = self.eps
        n = len(self.lr_table)
        self._froms = (C.c_uint64 * max(n, 1))(*[int(a) for a, _ in self.lr_table])
        self._vals = (C.c_double * max(n, 1))(*[float(b) for _, b in self.lr_table])
        h.lr_table_from = C.cast(self._froms, C.POINTER(C.c_uint64))
        h.lr_table_value = C.cast(self._vals, C.POINTER(C.c_double))
        h.lr_table_len = n
        return h

    def lr_at(self, t: int) -> float:
        """OptimizerHyper::lr_at, optim.cpp:50-57."""
        out = C.c_double()
        check(LIB.rw_lr_at(C.byref(self.to_c()), t, C.byref(out)))
        return out.value

    def validate(self) -> None:
        """OptimizerHyper::validate, optim.cpp:59-71."""
        check(LIB.rw_hyper_validate(C.byref(self.to_c())))


def flat_layout(sizes: Sequence[int], align: int = ALIGN_ELEMS) -> tuple[list[int], int]:
    """Offsets of each group in the flat buffers (groups start on `align`)."""
    offs, cur = [], 0
    for n in sizes:
        if n <= 0:
            raise RwError(1, "InvalidShape: zero extent")
        offs.append(cur)
        cur += (int(n) + align - 1) // align * align
    return offs, cur


def _stream_handle(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class DeviceState:
    """Flat device form of a list of ParamBlocks (optim.hpp:54-66).

    x, g, m, v are torch tensors owned here (caller-owned from the C ABI's
    point of view); the update-progress markers (t, updated) live in a
    device table inside the rw_state and are rewritten by the kernels.
    """

    def __init__(self, sizes: Sequence[int], dtype: torch.dtype = torch.float32,
                 device: int | torch.device | None = None, kind: int = ADAM,
                 with_vmax: bool = False,
                 align: int = ALIGN_ELEMS, host_resident: bool = False, stagger_bytes: int | None = None):
        if not torch.cuda.is_available():
            raise RwError(_lib.RW_CUDA_ERROR, "no CUDA device: the B200 path has no CPU fallback")
        if device is None:
            device = torch.cuda.current_device()
        dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.device = dev
        self.dtype = dtype
        self.rw_dtype = F64 if dtype == torch.float64 else F32
        if dtype not in (torch.float32, torch.float64):
            raise RwError(_lib.RW_INVALID_ARGUMENT, "state dtype must be float32 or float64")
        self.sizes = [int(n) for n in sizes]
        self.offsets, self.total = flat_layout(self.sizes, align)
        self.kind = kind
        uses_m = kind != SGD
        uses_v = kind in (ADAM, ADAMW, AMSGRAD, LAMB)
        groups = (rw_group * len(self.sizes))()
        for i, (o, n) in enumerate(zip(self.offsets, self.sizes)):
            groups[i].offset, groups[i].len, groups[i].t = o, n, 0
            groups[i].updated, groups[i].flags = 0, 0
        self._h = C.c_void_p()
        self.host_resident = host_resident
        if host_resident:  # layout + markers only: undo_from_host on host tensors (rw_state_create_host)
            self.x = self.g = self.m = self.v = self.vmax = None
            check(LIB.rw_state_create_host(C.byref(self._h), self.rw_dtype, self.total, groups,
                                           len(self.sizes), dev.index or 0))
            return
        uses_w = with_vmax or kind == AMSGRAD
        if stagger_bytes is None:
            alloc = lambda: torch.zeros(max(self.total, 1), dtype=dtype, device=dev)  # noqa: E731
        else:
            # one slab, buffer k starting k x (buffer bytes + stagger) in: the
            # streams the kernels read side by side (x[i], g[i], m[i], v[i])
            # are not a power-of-two distance apart in the physical address space
            es = torch.tensor([], dtype=dtype).element_size()
            pitch = (max(self.total, 1) * es + int(stagger_bytes) + 255) // 256 * 256 // es
            nbuf = 2 + int(uses_m) + int(uses_v) + int(uses_w)
            self._slab = torch.zeros(pitch * nbuf, dtype=dtype, device=dev)
            views = iter(self._slab[k * pitch:k * pitch + max(self.total, 1)] for k in range(nbuf))
            alloc = lambda: next(views)  # noqa: E731
        self.x = alloc()
        self.g = alloc()
        self.m = alloc() if uses_m else None
        self.v = alloc() if uses_v else None
        self.vmax = alloc() if uses_w else None
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        check(LIB.rw_state_create(C.byref(self._h), self.rw_dtype, ptr(self.x), ptr(self.g),
                                  ptr(self.m), ptr(self.v), ptr(self.vmax), self.total, groups,
                                  len(self.sizes), dev.index or 0))

    # ---- lifetime ----
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            LIB.rw_state_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def num_groups(self) -> int:
        return len(self.sizes)

    def view(self, which: str, i: int) -> torch.Tensor:
        buf = getattr(self, which)
        return buf[self.offsets[i]:self.offsets[i] + self.sizes[i]]

    def update_order(self) -> list[int]:
        """apply_layerwise_updates order: reverse layer order."""
        return list(range(self.num_groups - 1, -1, -1))

    # ---- the operator API (optim.hpp:71-76) ----
    def step(self, hyper: OptimizerHyper, ids: Iterable[int] | None = None,
             grad: torch.Tensor | None = None, stop_after: int | None = None, stream=None) -> None:
        """optimizer_step over groups `ids` (update order); grad in the flat layout."""
        ids = self.update_order() if ids is None else list(ids)
        arr = (C.c_uint32 * max(len(ids), 1))(*ids)
        gp = None
        if grad is not None:
            if grad.numel() < self.total or grad.dtype != self.dtype or grad.device != self.device:
                raise RwError(2, "ShapeMismatch: gradient shape does not match block")
            gp = C.c_void_p(grad.data_ptr())
        k = 0xFFFFFFFF if stop_after is None else int(stop_after)
        check(LIB.rw_optimizer_step(self._h, C.byref(hyper.to_c()), arr, len(ids), gp, k,
                                    C.c_void_p(_stream_handle(stream))))

    def undo(self, hyper: OptimizerHyper, ids: Iterable[int] | None = None, stream=None) -> None:
        """optimizer_undo over groups `ids`."""
        ids = self.update_order() if ids is None else list(ids)
        arr = (C.c_uint32 * max(len(ids), 1))(*ids)
        check(LIB.rw_optimizer_undo(self._h, C.byref(hyper.to_c()), arr, len(ids),
                                    C.c_void_p(_stream_handle(stream))))

    def undo_from_host(self, hyper: OptimizerHyper, host: dict, out: dict | None = None,
                       ids: Iterable[int] | None = None, slice_elems: int = 0, stream=None) -> None:
        """optimizer_undo of a state held in (pinned) host tensors host["x"/"g"/"m"/"v"]
        (this state's flat layout); results into out[...] (default: in place).
        H2D, undo and D2H are pipelined per slice of groups (rw_optimizer_undo_host)."""
        ids = self.update_order() if ids is None else list(ids)
        arr = (C.c_uint32 * max(len(ids), 1))(*ids)
        out = host if out is None else out
        for k, t in list(host.items()) + list(out.items()):
            if t is not None and (t.numel() < self.total or t.dtype != self.dtype or t.is_cuda):
                raise RwError(2, f"ShapeMismatch: host buffer {k} must be a {self.dtype} CPU tensor of "
                                 f">= {self.total} elements")
        p = lambda d, k: C.c_void_p(d[k].data_ptr()) if d.get(k) is not None else None  # noqa: E731
        check(LIB.rw_optimizer_undo_host(self._h, C.byref(hyper.to_c()), arr, len(ids), p(host, "x"),
                                         p(host, "g"), p(host, "m"), p(host, "v"), p(out, "x"), p(out, "m"),
                                         p(out, "v"), int(slice_elems), C.c_void_p(_stream_handle(stream))))

    def check_finite(self, stream=None) -> None:
        """Raise NumericalError if the last step/undo produced a non-finite value."""
        check(LIB.rw_state_check(self._h, C.c_void_p(_stream_handle(stream))))

    def clear_updated(self, ids: Iterable[int] | None = None, stream=None) -> None:
        ids = list(range(self.num_groups)) if ids is None else list(ids)
        arr = (C.c_uint32 * max(len(ids), 1))(*ids)
        check(LIB.rw_clear_updated(self._h, arr, len(ids), C.c_void_p(_stream_handle(stream))))

    def markers(self, stream=None) -> list[tuple[int, int]]:
        """(t, updated) per group, read from the device table."""
        g = self.read_groups(stream)
        return [(int(r.t), int(r.updated)) for r in g]

    def read_groups(self, stream=None):
        out = (rw_group * self.num_groups)()
        check(LIB.rw_state_read_groups(self._h, out, C.c_void_p(_stream_handle(stream))))
        return out

    def write_markers(self, markers: Sequence[tuple[int, int]], stream=None) -> None:
        g = self.read_groups(stream)
        for r, (t, u) in zip(g, markers):
            r.t, r.updated, r.flags = int(t), int(u), 0
        check(LIB.rw_state_write_groups(self._h, g, C.c_void_p(_stream_handle(stream))))

    def saved_scalars(self, i: int, stream=None) -> list[float]:
        """LAMB trust-ratio stack of group i, bottom -> top (optim.cpp:216)."""
        buf = (C.c_double * TRUST_DEPTH)()
        cnt = C.c_uint32()
        check(LIB.rw_state_saved_scalars(self._h, i, buf, TRUST_DEPTH, C.byref(cnt),
                                         C.c_void_p(_stream_handle(stream))))
        return list(buf[:cnt.value])

    def set_saved_scalars(self, i: int, vals: Sequence[float], stream=None) -> None:
        arr = (C.c_double * max(len(vals), 1))(*vals)
        check(LIB.rw_state_set_saved_scalars(self._h, i, arr, len(vals), C.c_void_p(_stream_handle(stream))))

    @property
    def handle(self) -> C.c_void_p:
        return self._h


def seeded_fill_(out: torch.Tensor, seed: int, offset: int = 0, stream=None) -> torch.Tensor:
    """Device seeded_fill (tensor.cpp:94-103) into a flat float32/float64 tensor."""
    dt = F64 if out.dtype == torch.float64 else F32
    check(LIB.rw_seeded_fill(dt, C.c_void_p(out.data_ptr()), out.numel(), seed, offset,
                             C.c_void_p(_stream_handle(stream))))
    return out


def derive_seed(base: int, parts: Sequence[int]) -> int:
    """derive_seed, tensor.cpp:76-83."""
    arr = (C.c_uint64 * max(len(parts), 1))(*parts)
    return int(LIB.rw_derive_seed(base, arr, len(parts)))


def ordered_sum(tensors: Sequence[torch.Tensor], out: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
    """ordered_sum (tensor.cpp:105-117) on the device, left to right."""
    if not tensors:
        raise RwError(3, "EmptyInput: ordered_sum of nothing")
    n = tensors[0].numel()
    for t in tensors:
        if t.numel() != n or t.dtype != tensors[0].dtype:
            raise RwError(2, "ShapeMismatch: ordered_sum shapes differ")
    out = torch.empty_like(tensors[0]) if out is None else out
    dt = F64 if out.dtype == torch.float64 else F32
    ptrs = (C.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    check(LIB.rw_ordered_sum(dt, ptrs, len(tensors), n, C.c_void_p(out.data_ptr()),
                             C.c_void_p(_stream_handle(stream))))
    return out
