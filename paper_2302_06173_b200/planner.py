"""Selective-logging policy (planner.cpp is absent from the
reference).  Thin Python mirror over the C++ implementation in
csrc/resolver_planner.cpp, keeping the SPEC operation names."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

from ._lib import LIB, check


@dataclass
class GroupPlan:
    """GroupPlan: contiguous machine groups + estimates."""

    groups: list[list[int]]
    storage: float    # M(G) = T * sum of inter-group boundary bytes
    recovery: float   # expected recovery seconds per lost iteration


def _darr(xs):
    xs = list(xs)
    return (C.c_double * max(len(xs), 1))(*xs)


def group_machines(R: Sequence[float], M: Sequence[float], B: float, T: float, M_max: float,
                   parallel: bool = False) -> GroupPlan:
    """group_machines(profile): greedy adjacent merge by min dR/dM."""
    N = len(R)
    gof = (C.c_uint32 * max(N, 1))()
    ng = C.c_uint32()
    st, rc = C.c_double(), C.c_double()
    check(LIB.rw_group_machines(N, _darr(R), _darr(M), B, T, M_max, int(parallel), gof,
                                C.byref(ng), C.byref(st), C.byref(rc)))
    groups: list[list[int]] = [[] for _ in range(ng.value)]
    for i in range(N):
        groups[gof[i]].append(i)
    return GroupPlan(groups, st.value, rc.value)


def recovery_time_estimate(R, M, B, groups, lost_iterations: float, parallel: bool = False) -> float:
    """recovery_time_estimate(plan, lost_iterations)."""
    N = len(R)
    gof = (C.c_uint32 * max(N, 1))()
    for gi, g in enumerate(groups):
        for mach in g:
            gof[mach] = gi
    out = C.c_double()
    check(LIB.rw_recovery_time_estimate(N, _darr(R), _darr(M), B, int(parallel), gof,
                                        lost_iterations, C.byref(out)))
    return out.value


def logging_worthwhile(bytes_per_iteration: float, pcie_bytes_per_s: float, p: int, m: int,
                       iteration_time_s: float) -> tuple[bool, float, float]:
    """logging_worthwhile -> (worthwhile, transfer_s, bubble_s)."""
    w = C.c_int32()
    tr, bb = C.c_double(), C.c_double()
    check(LIB.rw_logging_worthwhile(bytes_per_iteration, pcie_bytes_per_s, p, m, iteration_time_s,
                                    C.byref(w), C.byref(tr), C.byref(bb)))
    return bool(w.value), tr.value, bb.value


def boundary_elems(micro_batch: int, hidden: int, seq: int) -> int:
    """Elements per logged boundary message: micro_batch x hidden x seq (PAPER §5.4)."""
    return micro_batch * hidden * seq


def bubble_ratio(p: int, m: int) -> tuple[int, int]:
    """bubble_ratio (schedule.cpp:86-93) as an exact reduced fraction."""
    a, b = C.c_int64(), C.c_int64()
    check(LIB.rw_bubble_ratio(p, m, C.byref(a), C.byref(b)))
    return a.value, b.value
