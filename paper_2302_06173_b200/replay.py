"""Logging-based replay on the B200.

Reference semantics (model.cpp; recovery.cpp is absent):
  * a Stage is `num_layers` affine+tanh layers (make_stage, model.cpp:32-54),
    params in blocks() order W0, b0, W1, b1, ... (model.cpp:12-20);
  * an iteration runs every micro-batch forward + backward, accumulates the
    per-micro-batch gradients in ascending micro-batch order (accumulate_grads,
    model.cpp:158-172) and then steps every block in reverse layer order
    (apply_layerwise_updates);
  * recover_replay: the replacement loads the checkpoint and
    re-executes its stages feeding the logged inbound activations / gradients
    in timestamp order, applying the optimizer steps identically;
  * recover_parallel: helper h replays micro-batches
    {mb : mb mod d == h}; gradients are merged in ascending mb order (bit-exact
    equivalence with sequential replay), then one step.

Device mapping: fp32 master state (DeviceState, fused step kernels) + bf16
weight shadows; bf16 activations; tcgen05 GEMMs with fused epilogues
(csrc/umma_gemm.cuh).  Everything is deterministic, so a replay equals the
GPU ghost run bit for bit; against the fp64 reference it is tolerance-matched.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Sequence

import torch

from ._lib import LIB, RwError, check
from .optim import DeviceState, OptimizerHyper, derive_seed, seeded_fill_

RW_BF16 = 2


class rw_stage_desc(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("_pad", C.c_int32), ("dims", C.POINTER(C.c_int64)),
                ("w", C.POINTER(C.c_void_p)), ("b", C.POINTER(C.c_void_p))]


_sig = {
    "rw_stage_forward": (C.c_int, [C.POINTER(rw_stage_desc), C.c_int64, C.POINTER(C.c_void_p), C.c_void_p]),
    "rw_stage_backward": (C.c_int, [C.POINTER(rw_stage_desc), C.c_int64, C.POINTER(C.c_void_p), C.c_void_p,
                                    C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int32,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rw_stage_backward_ex": (C.c_int, [C.POINTER(rw_stage_desc), C.c_int64, C.POINTER(C.c_void_p), C.c_void_p,
                                       C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_void_p), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]),
    "rw_stage_backward_ex2": (C.c_int, [C.POINTER(rw_stage_desc), C.c_int64, C.POINTER(C.c_void_p), C.c_void_p,
                                        C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_void_p), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_uint64, C.c_void_p]),
    "rw_mse_grad": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p]),
    "rw_cast_f32_to_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "rw_replay_set_sm_reserve": (C.c_int, [C.c_int32]),
    "rw_replay_set_gemm_engine": (C.c_int, [C.c_int32, C.c_int32]),
}
for _n, (_r, _a) in _sig.items():
    _f = getattr(LIB, _n)
    _f.restype, _f.argtypes = _r, _a


_FUSE_DB = os.environ.get("RW_FUSE_DB", "1") != "0"


def _sh(stream=None) -> C.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _p(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None else None)


def synth_inputs(seed: int, iteration: int, stream: int, rows: int, dim: int,
                 dtype=torch.bfloat16, device=None) -> torch.Tensor:
    """synth_inputs (model.cpp:190-193): seeded_fill of derive_seed(seed, {1, it, stream})."""
    out = torch.empty(rows, dim, dtype=dtype, device=device or torch.cuda.current_device())
    _fill(out, derive_seed(seed, [1, iteration, stream]))
    return out


def synth_targets(seed: int, iteration: int, stream: int, rows: int, dim: int, device=None) -> torch.Tensor:
    """synth_targets (model.cpp:195-198), fp32."""
    out = torch.empty(rows, dim, dtype=torch.float32, device=device or torch.cuda.current_device())
    _fill(out, derive_seed(seed, [2, iteration, stream]))
    return out


def _fill(t: torch.Tensor, seed: int):
    dt = {torch.float32: 0, torch.float64: 1, torch.bfloat16: RW_BF16}[t.dtype]
    check(LIB.rw_seeded_fill(dt, _p(t), t.numel(), seed, 0, _sh()))


class Stage:
    """One pipeline stage (model.hpp:24-39) living on one GPU."""

    def __init__(self, stage_id: int, input_dim: int, hidden_dim: int, output_dim: int, num_layers: int,
                 seed: int, kind: int, device=None, dims: Sequence[int] | None = None):
        """make_stage(stage_id, input_dim, hidden_dim, output_dim, num_layers, seed)
        (model.cpp:32-54).  `dims` (num_layers + 1 widths) generalises the
        uniform hidden width, e.g. MLP blocks 4096 -> 11008 -> 4096 -> ..."""
        if num_layers < 1:
            raise RwError(18, "InvalidConfig: stage needs >= 1 layer")
        self.stage_id = stage_id
        self.dims = [input_dim] + [hidden_dim] * (num_layers - 1) + [output_dim]
        if dims is not None:
            if len(dims) != num_layers + 1:
                raise RwError(2, "ShapeMismatch: dims must have num_layers + 1 entries")
            self.dims = [int(d) for d in dims]
        self.L = num_layers
        sizes = []
        for l in range(num_layers):
            sizes += [self.dims[l] * self.dims[l + 1], self.dims[l + 1]]
        self.state = DeviceState(sizes, dtype=torch.float32, kind=kind, device=device)
        dev = self.state.device
        self.device = dev
        # make_stage (model.cpp:45-50): W_l from derive_seed(seed,{id,l,0}), b_l from {id,l,1}
        for l in range(num_layers):
            seeded_fill_(self.state.view("x", 2 * l), derive_seed(seed, [stage_id, l, 0]))
            seeded_fill_(self.state.view("x", 2 * l + 1), derive_seed(seed, [stage_id, l, 1]))
        self.grad = torch.zeros_like(self.state.x)  # flat, same layout as the state
        self.w16 = [torch.empty(self.dims[l] * self.dims[l + 1], dtype=torch.bfloat16, device=dev)
                    for l in range(num_layers)]
        self.refresh_shadows()
        self._dims_c = (C.c_int64 * (num_layers + 1))(*self.dims)
        self._w_c = (C.c_void_p * num_layers)(*[w.data_ptr() for w in self.w16])
        self._b_c = (C.c_void_p * num_layers)(*[self.state.view("x", 2 * l + 1).data_ptr()
                                                for l in range(num_layers)])
        self._dw_c = (C.c_void_p * num_layers)(*[self.grad_view(2 * l).data_ptr() for l in range(num_layers)])
        self._db_c = (C.c_void_p * num_layers)(*[self.grad_view(2 * l + 1).data_ptr()
                                                 for l in range(num_layers)])
        self.desc = rw_stage_desc(num_layers, 0, self._dims_c, self._w_c, self._b_c)
        self._scratch: dict = {}

    # ---- buffers ----
    def grad_view(self, i: int) -> torch.Tensor:
        o, n = self.state.offsets[i], self.state.sizes[i]
        return self.grad[o:o + n]

    def grad_ptrs(self, flat: torch.Tensor):
        """dw/db pointer arrays into a flat fp32 buffer laid out like the state."""
        o = self.state.offsets
        dw = (C.c_void_p * self.L)(*[flat[o[2 * l]:].data_ptr() for l in range(self.L)])
        db = (C.c_void_p * self.L)(*[flat[o[2 * l + 1]:].data_ptr() for l in range(self.L)])
        return dw, db

    def refresh_shadows(self, stream=None):
        for l in range(self.L):
            w = self.state.view("x", 2 * l)
            check(LIB.rw_cast_f32_to_bf16(_p(w), _p(self.w16[l]), w.numel(), _sh(stream)))

    def new_acts(self, rows: int, x: torch.Tensor | None = None) -> list[torch.Tensor]:
        """Activation cache of one micro-batch; acts[0] aliases the input `x`
        when given (the stage only reads it), so no copy is made."""
        first = [x] if x is not None else [torch.empty(rows, self.dims[0], dtype=torch.bfloat16, device=self.device)]
        return first + [torch.empty(rows, d, dtype=torch.bfloat16, device=self.device) for d in self.dims[1:]]

    def _scr(self, rows: int):
        if rows not in self._scratch:
            mx = max(self.dims)
            # fp32 scratch: ceil(rows/32) partial rows, so the dgrad GEMMs form the db sums (ex2)
            self._scratch[rows] = (torch.empty(rows * mx, dtype=torch.bfloat16, device=self.device),
                                   torch.empty(rows * mx, dtype=torch.bfloat16, device=self.device),
                                   torch.empty(max(64, (rows + 31) // 32) * mx, dtype=torch.float32,
                                               device=self.device))
        return self._scratch[rows]

    # ---- model.cpp entry points ----
    def forward(self, acts: Sequence[torch.Tensor], stream=None) -> torch.Tensor:
        """forward_stage: acts[0] is the input; fills acts[1..L]; returns acts[L]."""
        rows = acts[0].shape[0]
        arr = (C.c_void_p * (self.L + 1))(*[a.data_ptr() for a in acts])
        check(LIB.rw_stage_forward(C.byref(self.desc), rows, arr, _sh(stream)))
        return acts[-1]

    def backward(self, acts: Sequence[torch.Tensor], grad_in: torch.Tensor, grad_out: torch.Tensor | None,
                 accumulate: bool, dw=None, db=None, stream=None, grad_in_is_dz: bool = False,
                 prev_y: torch.Tensor | None = None, fuse_db: bool | None = None) -> None:
        """backward_stage + ordered accumulation into self.grad (or dw/db arrays).
        prev_y / grad_in_is_dz fuse a group-internal stage boundary (see
        rw_stage_backward_ex): grad_out becomes the previous stage's dz.
        fuse_db: db column sums formed in the dgrad epilogues (rw_stage_backward_ex2);
        None = on unless RW_FUSE_DB=0 (A/B runs)."""
        if fuse_db is None:
            fuse_db = _FUSE_DB
        rows = acts[0].shape[0]
        arr = (C.c_void_p * (self.L + 1))(*[a.data_ptr() for a in acts])
        s0, s1, sf = self._scr(rows)
        check(LIB.rw_stage_backward_ex2(C.byref(self.desc), rows, arr, _p(grad_in), int(grad_in_is_dz),
                                        _p(grad_out), _p(prev_y), dw or self._dw_c, db or self._db_c,
                                        int(accumulate), _p(s0), _p(s1), _p(sf), sf.numel() if fuse_db else 0,
                                        _sh(stream)))

    def step(self, hyper: OptimizerHyper, grad: torch.Tensor | None = None, stream=None) -> None:
        """apply_layerwise_updates over this stage (reverse layer order), then
        the iteration-end flag clear and the bf16 shadow refresh."""
        self.state.step(hyper, grad=self.grad if grad is None else grad, stream=stream)
        self.state.clear_updated(stream=stream)
        self.refresh_shadows(stream)

    def snapshot(self) -> dict:
        """In-HBM checkpoint of the stage state (x, m, v, markers)."""
        return dict(x=self.state.x.clone(), m=None if self.state.m is None else self.state.m.clone(),
                    v=None if self.state.v is None else self.state.v.clone(), markers=self.state.markers())

    def restore(self, snap: dict) -> None:
        self.state.x.copy_(snap["x"])
        if snap["m"] is not None:
            self.state.m.copy_(snap["m"])
        if snap["v"] is not None:
            self.state.v.copy_(snap["v"])
        self.state.write_markers(snap["markers"])
        self.refresh_shadows()


def mse_grad(pred: torch.Tensor, target: torch.Tensor, micro_batches: int,
             loss: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """mse_loss gradient (model.cpp:174-188) on the device: bf16 grad, fp64 loss."""
    grad = torch.empty_like(pred)
    scratch = torch.empty(256, dtype=torch.float64, device=pred.device)
    check(LIB.rw_mse_grad(_p(pred), _p(target), pred.numel(), micro_batches, _p(grad), _p(loss), _p(scratch),
                          _sh(stream)))
    return grad


@dataclass
class BoundaryLog:
    """Upstream-backup log of the messages INTO a group of stages:
    the activation entering its first stage and the gradient entering its last
    stage, per (iteration, micro-batch), in timestamp order.  Held in HBM or in
    pinned host memory (north_star)."""

    acts: dict = field(default_factory=dict)    # (it, mb) -> tensor
    grads: dict = field(default_factory=dict)
    pinned: bool = False
    _pending: dict = field(default_factory=dict, repr=False)  # prefetched H2D copies
    _stream: object = field(default=None, repr=False)

    def put(self, kind: str, it: int, mb: int, t: torch.Tensor, sender: int = 0, receiver: int = 0) -> None:
        if self.pinned:
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            t = h
        else:
            t = t.clone()
        (self.acts if kind == "act" else self.grads)[(it, mb)] = t

    def prefetch(self, kind: str, it: int, mb: int, device) -> None:
        """Start the H2D copy of a host-resident record on a side stream, so it
        overlaps the replay compute (get() then only waits for it)."""
        if not self.pinned:
            return
        t = (self.acts if kind == "act" else self.grads).get((it, mb))
        key = (kind, it, mb)
        if t is None or t.device == device or key in self._pending:
            return
        if self._stream is None:
            self._stream = torch.cuda.Stream(device=device)
        with torch.cuda.stream(self._stream):
            dev_t = t.to(device, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(self._stream)
        self._pending[key] = (dev_t, ev)

    def get(self, kind: str, it: int, mb: int, device) -> torch.Tensor | None:
        hit = self._pending.pop((kind, it, mb), None)
        if hit is not None:  # prefetched: wait for its copy, keep the memory alive for this stream
            dev_t, ev = hit
            torch.cuda.current_stream().wait_event(ev)
            dev_t.record_stream(torch.cuda.current_stream())
            return dev_t
        d = self.acts if kind == "act" else self.grads
        t = d.get((it, mb))
        if t is None:
            return None
        return t.to(device, non_blocking=True) if t.device != device else t

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for d in (self.acts, self.grads) for t in d.values())


class _LoggerSink:
    """Adapts logstore.Logger to the BoundaryLog.put interface (machine = stage)."""

    def __init__(self, logger):
        self.lg = logger

    def put(self, kind: str, it: int, mb: int, t: torch.Tensor, sender: int = 0, receiver: int = 0) -> None:
        from .logstore import RW_LOG_ACTIVATION, RW_LOG_GRADIENT
        self.lg.log_send(t, sender, receiver, it, mb, RW_LOG_ACTIVATION if kind == "act" else RW_LOG_GRADIENT)


class Pipeline:
    """A p-stage pipeline on one GPU used as the failure-free "ghost run"
    (SPEC:510): same seeds, same kernels.  Logs the boundaries around a group of
    stages [g0, g1] while training (log_send at group boundaries)."""

    def __init__(self, p: int, dim: int, hidden: int, layers: int, rows: int, micro_batches: int, seed: int,
                 kind: int, hyper: OptimizerHyper, device=None):
        self.stages = [Stage(s, dim, hidden, dim, layers, seed, kind, device) for s in range(p)]
        self.p, self.dim, self.rows, self.m, self.seed, self.hyper = p, dim, rows, micro_batches, seed, hyper
        self.iteration = 0
        self.losses: list[float] = []

    def run_iteration(self, log_group: tuple[int, int] | None = None, log=None,
                      cuts: Sequence[int] | None = None, senders: dict | None = None) -> float:
        """One training iteration.  `log` is a BoundaryLog (in HBM / pinned) or a
        logstore.Logger (async D2H + SWFT chunk files); the messages into the
        group [g0, g1] are logged at send time (upstream backup).

        Machines: `cuts` lists the stages that begin a machine (stage s with a
        machine boundary between s-1 and s); every message that crosses a cut
        is logged by its SENDER's machine, senders[machine] being that
        machine's Logger / BoundaryLog (each machine keeps the
        messages it sent, so a failed machine's inbound traffic survives on
        its neighbours)."""
        wrap = lambda lg: lg if (lg is None or isinstance(lg, BoundaryLog)) else _LoggerSink(lg)  # noqa: E731
        route = None
        if cuts:
            cut_set = sorted(set(int(c) for c in cuts))
            machine_of = lambda st: sum(1 for c in cut_set if c <= st)  # noqa: E731
            sinks = {k: wrap(v) for k, v in (senders or {}).items()}
            route = (set(cut_set), machine_of, sinks)
        return self._run_iteration(log_group, wrap(log), route)

    def _run_iteration(self, log_group, log, route=None) -> float:
        it = self.iteration
        dev = self.stages[0].device
        loss = torch.zeros(1, dtype=torch.float64, device=dev)
        tot = 0.0
        for mb in range(self.m):  # timestamp order
            x = synth_inputs(self.seed, it, mb, self.rows, self.dim, device=dev)
            all_acts = []
            for s, st in enumerate(self.stages):
                acts = st.new_acts(self.rows, x)
                if log_group and log is not None and s == log_group[0] and s > 0:
                    log.put("act", it, mb, x, sender=s - 1, receiver=s)
                if route and s in route[0] and route[1](s - 1) in route[2]:
                    route[2][route[1](s - 1)].put("act", it, mb, x, sender=s - 1, receiver=s)
                x = st.forward(acts)
                all_acts.append(acts)
            tgt = synth_targets(self.seed, it, mb, self.rows, self.dim, device=dev)
            g = mse_grad(x, tgt, self.m, loss)
            tot += float(loss.item())
            for s in range(self.p - 1, -1, -1):
                if log_group and log is not None and s == log_group[1] and s < self.p - 1:
                    log.put("grad", it, mb, g, sender=s + 1, receiver=s)
                if route and (s + 1) in route[0] and route[1](s + 1) in route[2]:
                    route[2][route[1](s + 1)].put("grad", it, mb, g, sender=s + 1, receiver=s)
                gout = torch.empty(self.rows, self.dim, dtype=torch.bfloat16, device=dev) if s > 0 else None
                self.stages[s].backward(all_acts[s], g, gout, accumulate=mb > 0)
                g = gout
        for st in reversed(self.stages):  # every stage updates after the flush
            st.step(self.hyper)
        self.iteration += 1
        self.losses.append(tot / self.m)
        return tot / self.m


def replay_group(stages: Sequence[Stage], log: BoundaryLog, it0: int, it1: int, rows: int, micro_batches: int,
                 seed: int, hyper: OptimizerHyper, first: bool, last: bool, dim: int) -> int:
    """recover_replay of a contiguous group of stages from its
    checkpoint (already loaded) through iterations [it0, it1): replays every
    micro-batch in timestamp order from the logged inbound tensors (or the
    re-derived synthetic inputs / targets at the pipeline ends, which are never
    logged, model.cpp:190-198).  Returns the number of replayed iterations."""
    dev = stages[0].device
    for it in range(it0, it1):
        for mb in range(micro_batches):
            # host-resident logs: this micro-batch's gradient and the next one's
            # activation move while this micro-batch computes
            if not last:
                log.prefetch("grad", it, mb, dev)
            if not first:
                nxt = (it, mb + 1) if mb + 1 < micro_batches else (it + 1, 0)
                log.prefetch("act", it, mb, dev)
                log.prefetch("act", nxt[0], nxt[1], dev)
            if first:
                x = synth_inputs(seed, it, mb, rows, dim, device=dev)
            else:
                x = log.get("act", it, mb, dev)
                if x is None:
                    raise RwError(14, f"MissingLogData: activation ({it}, {mb})")
            all_acts = []
            for st in stages:
                acts = st.new_acts(rows, x)
                x = st.forward(acts)
                all_acts.append(acts)
            if last:
                g = mse_grad(x, synth_targets(seed, it, mb, rows, dim, device=dev), micro_batches)
            else:
                g = log.get("grad", it, mb, dev)
                if g is None:
                    raise RwError(14, f"MissingLogData: gradient ({it}, {mb})")
            # group-internal boundaries stay on this GPU: stage k's first-layer
            # dgrad emits stage k-1's dz directly (bit-identical to the wire
            # round trip + dtanh of the original run)
            for k in range(len(stages) - 1, -1, -1):
                gout = torch.empty(rows, stages[k].dims[0], dtype=torch.bfloat16, device=dev) if k > 0 else None
                stages[k].backward(all_acts[k], g, gout, accumulate=mb > 0, grad_in_is_dz=k < len(stages) - 1,
                                   prev_y=all_acts[k - 1][-1] if k > 0 else None)
                g = gout
        for st in reversed(stages):
            st.step(hyper)
    log._pending.clear()  # a prefetch past the replayed range is not needed
    return it1 - it0


def parallel_assignment(m: int, d: int) -> list[list[int]]:
    """helper h replays micro-batches {mb : mb mod d == h}."""
    return [[mb for mb in range(m) if mb % d == h] for h in range(d)]


def helper_pass(stages: Sequence[Stage], log: BoundaryLog, it: int, mbs: Sequence[int], rows: int,
                micro_batches: int, seed: int, first: bool, last: bool, dim: int, on_stage_done=None) -> dict:
    """One helper's share of iteration `it`: forward + backward of its
    micro-batches, each into its OWN flat gradient buffers (one per stage), so
    the merge can restore the ascending-mb order exactly.  on_stage_done(k,
    {mb: buffer}) fires as soon as stage k's gradients of every micro-batch of
    this helper are complete (during the last micro-batch's backward), so the
    merge of stage k can overlap the backward of stages k-1..0."""
    dev = stages[0].device
    out = {}
    for n_mb, mb in enumerate(mbs):
        if not last:  # host-resident logs: overlap their H2D with this helper's compute
            log.prefetch("grad", it, mb, dev)
        if not first:
            log.prefetch("act", it, mb, dev)
            if n_mb + 1 < len(mbs):
                log.prefetch("act", it, mbs[n_mb + 1], dev)
        if first:
            x = synth_inputs(seed, it, mb, rows, dim, device=dev)
        else:
            x = log.get("act", it, mb, dev)
            if x is None:
                raise RwError(14, f"MissingLogData: activation ({it}, {mb})")
        all_acts = []
        for st in stages:
            acts = st.new_acts(rows, x)
            x = st.forward(acts)
            all_acts.append(acts)
        if last:
            g = mse_grad(x, synth_targets(seed, it, mb, rows, dim, device=dev), micro_batches)
        else:
            g = log.get("grad", it, mb, dev)
            if g is None:
                raise RwError(14, f"MissingLogData: gradient ({it}, {mb})")
        bufs = [torch.empty_like(st.grad) for st in stages]
        out[mb] = bufs
        for k in range(len(stages) - 1, -1, -1):
            gout = torch.empty(rows, stages[k].dims[0], dtype=torch.bfloat16, device=dev) if k > 0 else None
            dw, db = stages[k].grad_ptrs(bufs[k])
            stages[k].backward(all_acts[k], g, gout, accumulate=False, dw=dw, db=db,
                               grad_in_is_dz=k < len(stages) - 1, prev_y=all_acts[k - 1][-1] if k > 0 else None)
            g = gout
            if on_stage_done is not None and n_mb == len(mbs) - 1:
                on_stage_done(k, {b: out[b][k] for b in mbs})
    return out


def _shard_bounds(P: int, d: int) -> tuple[int, list[tuple[int, int]]]:
    chunk = ((P + d - 1) // d + 63) // 64 * 64
    return chunk, [(min(P, j * chunk), min(P, (j + 1) * chunk)) for j in range(d)]


def ordered_merge_start(bufs: dict, P: int, m: int, group=None, device=None):
    """Start the ordered merge of one stage's gradient over the d
    helpers: the flat gradient is sharded over the ranks; every owner sends
    shard j of each of its micro-batches to rank j in ONE grouped batch of
    point-to-point transfers (all links busy at once, no packing copies).
    Asynchronous: returns a handle for ordered_merge_finish."""
    import torch.distributed as dist
    d, rank = dist.get_world_size(group), dist.get_rank(group)
    glob = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)  # noqa: E731
    chunk, bnd = _shard_bounds(P, d)
    lo, hi = bnd[rank]
    dev = device if device is not None else (next(iter(bufs.values())).device if bufs else
                                              torch.device("cuda", torch.cuda.current_device()))
    recv, ops = {}, []
    for mb in range(m):
        owner = mb % d
        if owner == rank:
            for j in range(d):
                if j != rank and bnd[j][1] > bnd[j][0]:
                    ops.append(dist.P2POp(dist.isend, bufs[mb][bnd[j][0]:bnd[j][1]], glob(j), group))
        elif hi > lo:
            recv[mb] = torch.empty(hi - lo, dtype=torch.float32, device=dev)
            ops.append(dist.P2POp(dist.irecv, recv[mb], glob(owner), group))
    works = dist.batch_isend_irecv(ops) if ops else []
    return dict(works=works, recv=recv, bufs=bufs, P=P, m=m, group=group, chunk=chunk, lo=lo, hi=hi, d=d, dev=dev)


def ordered_merge_finish(h, summer=None) -> torch.Tensor:
    """Finish a merge: sum this rank's shard over micro-batches 0..m-1 in
    ascending order (ordered_sum, bit-identical to the sequential replay) and
    all-gather the merged shards into the full gradient.  `summer(parts, out)`
    replaces the device ordered_sum only in the CPU (gloo) tests of this
    bookkeeping, which pass the oracle's sum."""
    import torch.distributed as dist
    if summer is None:
        from .optim import ordered_sum as summer
    for w in h["works"]:
        w.wait()
    lo, hi, chunk, d = h["lo"], h["hi"], h["chunk"], h["d"]
    shard = torch.zeros(chunk, dtype=torch.float32, device=h["dev"])
    if hi > lo:
        parts = [h["recv"][mb] if mb in h["recv"] else h["bufs"][mb][lo:hi] for mb in range(h["m"])]
        summer(parts, out=shard[:hi - lo])
    if dist.get_backend(h["group"]) == "nccl":
        full = torch.empty(chunk * d, dtype=torch.float32, device=h["dev"])
        dist.all_gather_into_tensor(full, shard, group=h["group"])
    else:  # gloo (CPU tests): list form
        parts = [torch.empty_like(shard) for _ in range(d)]
        dist.all_gather(parts, shard, group=h["group"])
        full = torch.cat(parts)
    return full[:h["P"]]


def ordered_merge(per_mb: dict, k: int, m: int, group=None) -> torch.Tensor:
    """Merged gradient of stage k: ordered_sum over micro-batches 0..m-1
    (SPEC:538).  Without a process group every micro-batch is local; with one,
    sharded point-to-point exchange + local ordered sum + all-gather (every rank
    then steps redundantly and identically)."""
    from .optim import ordered_sum
    import torch.distributed as dist
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return ordered_sum([per_mb[mb][k] for mb in range(m)])
    any_buf = next(iter(per_mb.values()))[k]
    return ordered_merge_finish(ordered_merge_start({mb: b[k] for mb, b in per_mb.items()}, any_buf.numel(), m,
                                                    group))


_MERGE_GROUPS: dict = {}


def _merge_group(max_ctas: int):
    """A NCCL communicator for the merges whose kernels use at most
    `max_ctas` CTAs (= the SMs the replay GEMMs leave free)."""
    import torch.distributed as dist
    key = (dist.get_world_size(), max_ctas)
    if key not in _MERGE_GROUPS:
        opts = dist.ProcessGroupNCCL.Options()
        opts.config.max_ctas = max_ctas
        opts.config.min_ctas = 1
        _MERGE_GROUPS[key] = dist.new_group(backend="nccl", pg_options=opts)
    return _MERGE_GROUPS[key]


_CE_MERGERS: dict = {}


def recover_parallel(stages: Sequence[Stage], log: BoundaryLog, it0: int, it1: int, rows: int,
                     micro_batches: int, seed: int, hyper: OptimizerHyper, first: bool, last: bool, dim: int,
                     group=None, rank: int = 0, d: int = 1, merge: str = "auto", overlap: bool = False,
                     reserve_sms: int = 8) -> int:
    """recover_parallel for this helper rank.

    merge="copy_engine" (auto with NCCL on one node): each stage's shards leave
    over the DMA engines as soon as its gradients are complete, overlapping the
    backward of the earlier stages without taking SMs from the GEMMs
    (merge.CopyEngineMerger); the ordered sums, the gather and the steps follow.
    merge="nccl": grouped point-to-point exchange after the pass (or, with
    overlap=True, during it on a communicator capped at `reserve_sms` CTAs
    while the GEMMs leave that many SMs free: measured slower, N=4 220 vs
    203 ms/iteration).  Every path sums in ascending micro-batch order, so all
    are bit-identical to the sequential replay."""
    import torch.distributed as dist
    assign = parallel_assignment(micro_batches, d)
    distributed = group is not None or (dist.is_available() and dist.is_initialized())
    nccl = distributed and dist.get_backend(group) == "nccl"
    if merge == "auto":
        merge = "copy_engine" if (nccl and dist.get_world_size(group) <= torch.cuda.device_count()) else "nccl"
    if distributed and merge == "copy_engine":
        return _recover_parallel_ce(stages, log, it0, it1, rows, micro_batches, seed, hyper, first, last, dim,
                                    group, rank, assign)
    use_overlap = (nccl and overlap and group is None and reserve_sms > 0)
    mgroup = _merge_group(reserve_sms) if use_overlap else group
    if use_overlap:
        check(LIB.rw_replay_set_sm_reserve(reserve_sms))
    try:
        for it in range(it0, it1):
            handles = {}

            def start(k, bufs):
                handles[k] = ordered_merge_start(bufs, stages[k].grad.numel(), micro_batches, mgroup)

            per_mb = helper_pass(stages, log, it, assign[rank], rows, micro_batches, seed, first, last, dim,
                                 on_stage_done=start if use_overlap else None)
            if distributed:
                for k in range(len(stages) - 1, -1, -1):  # same order on every rank
                    if k not in handles:
                        start(k, {mb: per_mb[mb][k] for mb in assign[rank]})
            for k, st in enumerate(stages):
                if distributed:
                    merged = ordered_merge_finish(handles[k])
                else:
                    merged = ordered_merge(per_mb, k, micro_batches, None)
                st.step(hyper, grad=merged)
    finally:
        if use_overlap:
            check(LIB.rw_replay_set_sm_reserve(0))
    return it1 - it0


def _recover_parallel_ce(stages, log, it0, it1, rows, micro_batches, seed, hyper, first, last, dim, group, rank,
                         assign) -> int:
    from .merge import CopyEngineMerger
    import torch.distributed as dist
    key = (tuple(st.grad.numel() for st in stages), micro_batches, dist.get_world_size(group), id(group))
    if key not in _CE_MERGERS:
        _CE_MERGERS[key] = CopyEngineMerger(key[0], micro_batches, group)
    mg = _CE_MERGERS[key]
    for it in range(it0, it1):
        mg.begin_iteration()
        pending = {}

        def ship(k, bufs):
            # scatter + (queued behind the peers' counters) reduce and gather of
            # stage k, overlapping the backward of stages k-1..0
            mg.scatter(k, bufs)
            pending[k] = mg.reduce_gather(k, bufs, wait=False)

        per_mb = helper_pass(stages, log, it, assign[rank], rows, micro_batches, seed, first, last, dim,
                             on_stage_done=ship)
        for k in range(len(stages) - 1, -1, -1):  # a helper without micro-batches still signals
            if k not in pending:
                ship(k, {mb: per_mb[mb][k] for mb in assign[rank]})
        for k, st in enumerate(stages):
            merged, ev = pending[k]
            torch.cuda.current_stream().wait_event(ev)
            st.step(hyper, grad=merged)
    return it1 - it0
