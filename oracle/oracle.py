"""ORACLE — test infrastructure, not product code.

ctypes access to
  * ``oracle/_ref/librewind_ref.so`` — the UNMODIFIED reference library built
    from /root/reference by oracle/Makefile (the "reference itself run here"),
  * ``oracle/_build/liboracle.so``  — our plain-C restatement (restate.c) in
    fp64 (pinned bit-exact against _ref) and fp32 (the bit-exact target of the
    CUDA fp32 kernels),
plus pure-Python restatements of the SPEC-only pieces (no reference source
exists for them: recovery.cpp / planner.cpp are missing):
consensus_iteration + apply_undo, group_machines /
recovery_time_estimate / brute_force_group_oracle,
logging_worthwhile, parallel micro-batch assignment
(SPEC:511-519).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import itertools
import math
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "librewind_ref.so"
RESTATE_SO = HERE / "_build" / "liboracle.so"

SGD, SGDM, ADAM, ADAMW, LAMB, AMSGRAD = range(6)
ERR = ["InvalidShape", "ShapeMismatch", "EmptyInput", "NumericalError", "NonInvertibleHyper",
       "NotInvertible", "NothingToUndo", "AlreadyUpdated", "MissingActivation", "ChannelBroken",
       "InvalidInjection", "NotFailed", "StorageError", "MissingLogData", "CorruptLog",
       "NoCheckpoint", "NoReplica", "InvalidConfig", "TooLarge"]

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = ERR[status - 1] if 1 <= status <= 19 else "Unknown"
        super().__init__(msg)


class ref_hyper_c(C.Structure):
    _fields_ = [("kind", C.c_int), ("lr", C.c_double), ("weight_decay", C.c_double),
                ("momentum", C.c_double), ("dampening", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("require_invertible", C.c_int),
                ("n_lr_table", C.c_int), ("lr_from", C.POINTER(C.c_uint64)),
                ("lr_value", _dp)]


class or_hyper(C.Structure):
    _fields_ = [("kind", C.c_int), ("lr", C.c_double), ("weight_decay", C.c_double),
                ("momentum", C.c_double), ("dampening", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("n_lr_table", C.c_int),
                ("lr_from", C.POINTER(C.c_uint64)), ("lr_value", _dp)]


class or_scalars(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("eta", "c1", "c2", "wd", "mu", "one_m_damp", "b1", "b2",
                                          "one_m_b1", "one_m_b2", "eps", "denom")]


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _fptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_fp)


def _hyper_fields(h) -> dict:
    """Accept any object with the OptimizerHyper field names."""
    get = (lambda k, d=None: h.get(k, d)) if isinstance(h, dict) else (
        lambda k, d=None: getattr(h, k, d))
    return dict(kind=get("kind", SGD), lr=get("lr", 0.01), weight_decay=get("weight_decay", 0.0),
                momentum=get("momentum", 0.9), dampening=get("dampening", 0.0),
                beta1=get("beta1", 0.9), beta2=get("beta2", 0.999), eps=get("eps", 1e-8),
                require_invertible=bool(get("require_invertible", False)),
                lr_table=list(get("lr_table", []) or []))


# ---------------------------------------------------------------- reference
class Ref:
    """The reference library itself (oracle/_ref)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(str(path))
        vp, sz, u64, i = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int
        P = C.POINTER
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_block_make": (vp, [P(sz), i, u64]),
            "ref_block_free": (None, [vp]),
            "ref_block_size": (sz, [vp]),
            "ref_block_set": (None, [vp, _dp, _dp, _dp, _dp, u64, i]),
            "ref_block_get": (None, [vp, _dp, _dp, _dp, _dp, P(u64), P(i)]),
            "ref_block_saved_scalars": (i, [vp, _dp, i]),
            "ref_optimizer_step": (i, [vp, _dp, P(sz), i, P(ref_hyper_c)]),
            "ref_optimizer_undo": (i, [vp, P(ref_hyper_c)]),
            "ref_invertibility_check": (i, [i]),
            "ref_lr_at": (i, [P(ref_hyper_c), u64, _dp]),
            "ref_validate": (i, [P(ref_hyper_c)]),
            "ref_optimizer_from_name": (i, [C.c_char_p]),
            "ref_mix64": (u64, [u64]),
            "ref_derive_seed": (u64, [u64, P(u64), i]),
            "ref_seeded_fill": (i, [P(sz), i, u64, _dp]),
            "ref_ordered_sum": (i, [P(_dp), P(sz), i, _dp]),
            "ref_l2_norm": (i, [_dp, sz, _dp]),
            "ref_crc32": (C.c_uint32, [C.c_char_p, sz]),
            "ref_fnv1a64": (u64, [C.c_char_p, sz]),
            "ref_bubble_ratio": (i, [i, i, P(C.c_longlong), P(C.c_longlong)]),
            "ref_build_1f1b_schedule": (i, [i, i, P(i), P(i), i, P(i)]),
            "ref_schedule_grid": (i, [i, i, C.c_char_p, sz]),
            "ref_count_bubbles": (C.c_longlong, [i, i]),
            "ref_stage_make": (vp, [i, sz, sz, sz, i, u64]),
            "ref_stage_free": (None, [vp]),
            "ref_stage_nblocks": (i, [vp]),
            "ref_stage_block": (vp, [vp, i]),
            "ref_forward_stage": (i, [vp, _dp, sz, sz, C.c_uint32, _dp]),
            "ref_backward_stage": (i, [vp, _dp, sz, sz, C.c_uint32, _dp, P(_dp)]),
            "ref_mse_loss": (i, [_dp, _dp, sz, sz, sz, _dp, _dp]),
            "ref_synth_inputs": (i, [u64, u64, u64, sz, sz, _dp]),
            "ref_synth_targets": (i, [u64, u64, u64, sz, sz, _dp]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a

    def _chk(self, st: int):
        if st:
            raise RefError(st, self.L.ref_last_error().decode())

    @staticmethod
    def hyper(h) -> ref_hyper_c:
        f = _hyper_fields(h)
        c = ref_hyper_c()
        c.kind, c.lr, c.weight_decay = f["kind"], f["lr"], f["weight_decay"]
        c.momentum, c.dampening, c.beta1, c.beta2 = f["momentum"], f["dampening"], f["beta1"], f["beta2"]
        c.eps, c.require_invertible = f["eps"], int(f["require_invertible"])
        n = len(f["lr_table"])
        c._f = (C.c_uint64 * max(n, 1))(*[a for a, _ in f["lr_table"]])
        c._v = (C.c_double * max(n, 1))(*[b for _, b in f["lr_table"]])
        c.n_lr_table, c.lr_from, c.lr_value = n, c._f, c._v
        return c

    # ---- ParamBlock handle ----
    def block(self, n: int, seed: int = 0) -> "RefBlock":
        return RefBlock(self, (n,), seed)

    def seeded_fill(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        shp = (C.c_size_t * 1)(n)
        self._chk(self.L.ref_seeded_fill(shp, 1, seed, _dptr(out)))
        return out

    def derive_seed(self, base: int, parts) -> int:
        arr = (C.c_uint64 * max(len(parts), 1))(*parts)
        return int(self.L.ref_derive_seed(base, arr, len(parts)))

    def ordered_sum(self, arrays) -> np.ndarray:
        arrays = [np.ascontiguousarray(a, np.float64) for a in arrays]
        ptrs = (_dp * max(len(arrays), 1))(*[_dptr(a) for a in arrays])
        lens = (C.c_size_t * max(len(arrays), 1))(*[a.size for a in arrays])
        out = np.empty(arrays[0].size if arrays else 0, np.float64)
        self._chk(self.L.ref_ordered_sum(ptrs, lens, len(arrays), _dptr(out) if out.size else None))
        return out

    def l2_norm(self, a) -> float:
        a = np.ascontiguousarray(a, np.float64)
        out = C.c_double()
        self._chk(self.L.ref_l2_norm(_dptr(a), a.size, C.byref(out)))
        return out.value

    def crc32(self, b: bytes) -> int:
        return int(self.L.ref_crc32(b, len(b)))

    def bubble_ratio(self, p: int, m: int) -> tuple[int, int]:
        a, b = C.c_longlong(), C.c_longlong()
        self._chk(self.L.ref_bubble_ratio(p, m, C.byref(a), C.byref(b)))
        return a.value, b.value

    def schedule(self, p: int, m: int):
        cap = 2 * (m + p) + 8
        kinds = (C.c_int * (p * cap))()
        mbs = (C.c_int * (p * cap))()
        slots = C.c_int()
        self._chk(self.L.ref_build_1f1b_schedule(p, m, kinds, mbs, cap, C.byref(slots)))
        n = slots.value
        return [[(kinds[s * cap + i], mbs[s * cap + i]) for i in range(n)] for s in range(p)]

    def schedule_grid(self, p: int, m: int) -> str:
        buf = C.create_string_buffer(1 << 16)
        self._chk(self.L.ref_schedule_grid(p, m, buf, len(buf)))
        return buf.value.decode()

    def lr_at(self, h, t: int) -> float:
        out = C.c_double()
        self._chk(self.L.ref_lr_at(C.byref(self.hyper(h)), t, C.byref(out)))
        return out.value


class RefBlock:
    """A reference ParamBlock (optim.hpp:54-66) behind a handle."""

    def __init__(self, ref: Ref, shape, seed: int):
        self.ref = ref
        shp = (C.c_size_t * len(shape))(*shape)
        self.shape = tuple(shape)
        self.h = ref.L.ref_block_make(shp, len(shape), seed)
        if not self.h:
            raise RefError(1, ref.L.ref_last_error().decode())
        self.n = int(ref.L.ref_block_size(self.h))

    def __del__(self):
        try:
            self.ref.L.ref_block_free(self.h)
        except Exception:
            pass

    def set(self, x=None, g=None, m=None, v=None, t=0, updated=False):
        arrs = [None if a is None else np.ascontiguousarray(a, np.float64) for a in (x, g, m, v)]
        ps = [None if a is None else _dptr(a) for a in arrs]
        self.ref.L.ref_block_set(self.h, *ps, t, int(updated))

    def get(self):
        x, g, m, v = (np.empty(self.n) for _ in range(4))
        t, u = C.c_uint64(), C.c_int()
        self.ref.L.ref_block_get(self.h, _dptr(x), _dptr(g), _dptr(m), _dptr(v), C.byref(t), C.byref(u))
        return dict(x=x, g=g, m=m, v=v, t=t.value, updated=bool(u.value))

    def step(self, grad, h):
        grad = np.ascontiguousarray(grad, np.float64)
        shp = (C.c_size_t * len(self.shape))(*self.shape)
        self.ref._chk(self.ref.L.ref_optimizer_step(self.h, _dptr(grad), shp, len(self.shape),
                                                    C.byref(Ref.hyper(h))))

    def undo(self, h):
        self.ref._chk(self.ref.L.ref_optimizer_undo(self.h, C.byref(Ref.hyper(h))))

    def saved_scalars(self):
        buf = (C.c_double * 256)()
        n = self.ref.L.ref_block_saved_scalars(self.h, buf, 256)
        return list(buf[:n])


# ---------------------------------------------------------------- restatement
class Restate:
    """Our plain-C restatement (restate.c), fp64 and fp32."""

    def __init__(self, path: Path = RESTATE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(str(path))
        sz, u64 = C.c_size_t, C.c_uint64
        P = C.POINTER
        L.oracle_scalars.restype = C.c_int
        L.oracle_scalars.argtypes = [P(or_hyper), u64, C.c_int, P(or_scalars)]
        for suf, p in (("f64", _dp), ("f32", _fp)):
            for op in ("step", "undo"):
                f = getattr(L, f"oracle_{op}_{suf}")
                f.restype, f.argtypes = C.c_int, [C.c_int, P(or_scalars), p, p, p, p, sz]
            f = getattr(L, f"oracle_step_amsgrad_{suf}")
            f.restype, f.argtypes = C.c_int, [P(or_scalars), p, p, p, p, p, sz]
            f = getattr(L, f"oracle_ordered_sum_{suf}")
            f.restype, f.argtypes = None, [P(p), C.c_int, sz, p]
            f = getattr(L, f"oracle_seeded_fill_{suf}")
            f.restype, f.argtypes = None, [u64, sz, p]
        L.oracle_step_lamb_f64.restype = C.c_int
        L.oracle_step_lamb_f64.argtypes = [P(or_scalars), _dp, _dp, _dp, _dp, sz, _dp]
        L.oracle_undo_lamb_f64.restype = C.c_int
        L.oracle_undo_lamb_f64.argtypes = [P(or_scalars), C.c_double, _dp, _dp, _dp, _dp, sz]
        L.oracle_derive_seed.restype = u64
        L.oracle_derive_seed.argtypes = [u64, P(u64), C.c_int]

    @staticmethod
    def hyper(h) -> or_hyper:
        f = _hyper_fields(h)
        c = or_hyper()
        c.kind, c.lr, c.weight_decay = f["kind"], f["lr"], f["weight_decay"]
        c.momentum, c.dampening, c.beta1, c.beta2 = f["momentum"], f["dampening"], f["beta1"], f["beta2"]
        c.eps = f["eps"]
        n = len(f["lr_table"])
        c._f = (C.c_uint64 * max(n, 1))(*[a for a, _ in f["lr_table"]])
        c._v = (C.c_double * max(n, 1))(*[b for _, b in f["lr_table"]])
        c.n_lr_table, c.lr_from, c.lr_value = n, c._f, c._v
        return c

    def scalars(self, h, t_before: int, undo: bool) -> or_scalars:
        s = or_scalars()
        st = self.L.oracle_scalars(C.byref(self.hyper(h)), t_before, int(undo), C.byref(s))
        if st:
            raise RefError(st, "InvalidConfig: learning rate must be positive")
        return s

    def _arrs(self, dtype, *arrs):
        return [np.array(a, dtype=dtype, copy=True, order="C") for a in arrs]

    def step(self, kind, h, t_before, x, g, m, v, dtype=np.float64):
        """In place on copies; returns (x, m, v, nonfinite_flag)."""
        x, g, m, v = self._arrs(dtype, x, g, m, v)
        s = self.scalars(h, t_before, False)
        f = self.L.oracle_step_f64 if dtype == np.float64 else self.L.oracle_step_f32
        p = _dptr if dtype == np.float64 else _fptr
        fin = f(kind, C.byref(s), p(x), p(g), p(m), p(v), x.size)
        return x, m, v, bool(fin)

    def undo(self, kind, h, t_before, x, g, m, v, dtype=np.float64):
        x, g, m, v = self._arrs(dtype, x, g, m, v)
        s = self.scalars(h, t_before, True)
        f = self.L.oracle_undo_f64 if dtype == np.float64 else self.L.oracle_undo_f32
        p = _dptr if dtype == np.float64 else _fptr
        fin = f(kind, C.byref(s), p(x), p(g), p(m), p(v), x.size)
        return x, m, v, bool(fin)

    def step_amsgrad(self, h, t_before, x, g, m, v, vmax, dtype=np.float64):
        x, g, m, v, vmax = self._arrs(dtype, x, g, m, v, vmax)
        s = self.scalars(h, t_before, False)
        f = self.L.oracle_step_amsgrad_f64 if dtype == np.float64 else self.L.oracle_step_amsgrad_f32
        p = _dptr if dtype == np.float64 else _fptr
        fin = f(C.byref(s), p(x), p(g), p(m), p(v), p(vmax), x.size)
        return x, m, v, vmax, bool(fin)

    def ordered_sum(self, arrays, dtype=np.float64):
        arrays = [np.ascontiguousarray(a, dtype) for a in arrays]
        p, P = (_dptr, _dp) if dtype == np.float64 else (_fptr, _fp)
        ptrs = (P * len(arrays))(*[p(a) for a in arrays])
        out = np.empty(arrays[0].size, dtype)
        f = self.L.oracle_ordered_sum_f64 if dtype == np.float64 else self.L.oracle_ordered_sum_f32
        f(ptrs, len(arrays), out.size, p(out))
        return out

    def seeded_fill(self, n, seed, dtype=np.float64):
        out = np.empty(n, dtype)
        if dtype == np.float64:
            self.L.oracle_seeded_fill_f64(seed, n, _dptr(out))
        else:
            self.L.oracle_seeded_fill_f32(seed, n, _fptr(out))
        return out

    def derive_seed(self, base, parts):
        arr = (C.c_uint64 * max(len(parts), 1))(*parts)
        return int(self.L.oracle_derive_seed(base, arr, len(parts)))


# ------------------------------------------------- SPEC-only restatements
def consensus_iteration(iterations) -> int:
    """minimum over survivors."""
    return min(iterations)


def resolve(markers_per_rank, grad_ready_per_rank=None, invertible=True, policy="undo"):
    """Restatement of consensus + apply_undo with redo.

    markers_per_rank: list (ranks) of list (groups) of (t, updated).
    Returns (strategy, target, actions_per_rank) with actions "none"/"undo"/"redo".
    """
    ts = [t for r in markers_per_rank for t, _ in r]
    lo, hi = min(ts), max(ts)
    acts = [["none"] * len(r) for r in markers_per_rank]
    if hi == lo:
        return "None", lo, acts
    if hi > lo + 1:
        return "GlobalRollback", lo, acts
    undo_cost = max(sum(1 for t, _ in r if t == lo + 1) for r in markers_per_rank)
    if grad_ready_per_rank is None:
        grad_ready_per_rank = [[False] * len(r) for r in markers_per_rank]
    can_redo = all(gr for r, rdy in zip(markers_per_rank, grad_ready_per_rank)
                   for (t, _), gr in zip(r, rdy) if t == lo)
    redo_cost = max(sum(1 for t, _ in r if t == lo) for r in markers_per_rank)
    if policy == "min_cost" and invertible and can_redo:
        strat = "Redo" if redo_cost < undo_cost else "Undo"
    elif invertible:
        strat = "Undo"
    elif can_redo:
        strat = "Redo"
    else:
        strat = "GlobalRollback"
    target = lo + 1 if strat == "Redo" else lo
    for ri, r in enumerate(markers_per_rank):
        for gi, (t, _) in enumerate(r):
            if strat == "Undo" and t == lo + 1:
                acts[ri][gi] = "undo"
            if strat == "Redo" and t == lo:
                acts[ri][gi] = "redo"
    return strat, target, acts


def _weighted(size, R, N, parallel):
    r = R / math.floor(N / size) if parallel else R
    return size / N * r


def plan_cost(groups, R, M, B, T, N, parallel):
    """(storage M(G), expected recovery R per lost iteration) of a plan."""
    stor = 0.0
    rec = 0.0
    for gi, grp in enumerate(groups):
        r = 0.0
        for k, mach in enumerate(grp):
            r = r + R[mach]
            if k > 0:
                r = r + M[mach - 1] / B
        rec += _weighted(len(grp), r, N, parallel)
        if gi + 1 < len(groups):
            stor += M[grp[-1]]
    return T * stor, rec


def group_machines(R, M, B, T, M_max, parallel=False):
    """Greedy merge, restated in Python for the tests."""
    N = len(R)
    groups = [[i] for i in range(N)]
    Rg = list(R)

    def storage():
        return T * sum(M[g[-1]] for g in groups[:-1])

    while storage() > M_max and len(groups) > 1:
        best = None
        for i in range(len(groups) - 1):
            m = M[groups[i][-1]]
            merged = Rg[i] + Rg[i + 1] + m / B
            dR = (_weighted(len(groups[i]) + len(groups[i + 1]), merged, N, parallel)
                  - _weighted(len(groups[i]), Rg[i], N, parallel)
                  - _weighted(len(groups[i + 1]), Rg[i + 1], N, parallel))
            dM = T * m
            key = (0, dR / dM) if dM > 0 else (1, 0.0)
            if best is None or key < best[0]:
                best = (key, i)
        i = best[1]
        m = M[groups[i][-1]]
        Rg[i] = Rg[i] + Rg[i + 1] + m / B
        groups[i] = groups[i] + groups[i + 1]
        del groups[i + 1], Rg[i + 1]
    return groups


def brute_force_group_oracle(R, M, B, T, M_max, parallel=False):
    """min recovery over all 2^(N-1) contiguous partitions."""
    N = len(R)
    if N > 12:
        raise RefError(19, "TooLarge: N > 12")
    best = None
    for cuts in itertools.product([0, 1], repeat=N - 1):
        groups, cur = [], [0]
        for i, c in enumerate(cuts):
            if c:
                groups.append(cur)
                cur = [i + 1]
            else:
                cur.append(i + 1)
        groups.append(cur)
        stor, rec = plan_cost(groups, R, M, B, T, N, parallel)
        if stor <= M_max and (best is None or rec < best[0]):
            best = (rec, groups)
    return best[1] if best else [list(range(N))]


def logging_worthwhile(bytes_per_iteration, pcie_bw, p, m, iteration_time):
    """SPEC:594-602."""
    br = (p - 1) / (m + p - 1)
    transfer = bytes_per_iteration / pcie_bw
    bubble = br * iteration_time
    ok = transfer <= bubble and not (bytes_per_iteration > 0 and br == 0)
    return ok, transfer, bubble


def parallel_assignment(m: int, d: int):
    """helper h replays micro-batches {mb : mb mod d == h}."""
    return [[mb for mb in range(m) if mb % d == h] for h in range(d)]
