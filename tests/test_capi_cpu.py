"""C-ABI library checks that need no GPU: it loads, exports every symbol the
header declares, host-only entry points agree with the reference/oracle, and
GPU entry points fail loudly (no CPU fallback) when no device is visible."""
import ctypes as C
import random

import numpy as np
import pytest

from paper_2302_06173_b200 import _lib
from paper_2302_06173_b200._lib import LIB, RwError, check, rw_group, rw_hyper, rw_resolve_summary
from paper_2302_06173_b200.optim import OptimizerHyper, flat_layout, invertibility_check
from paper_2302_06173_b200 import planner


def test_exports_every_declared_symbol():
    declared = _lib.declared_functions()
    assert len(declared) >= 25
    exported = _lib.library_exports()
    missing = [f for f in declared if f not in exported]
    assert not missing, missing


def test_status_codes_mirror_reference_err(ref):
    # status = 1 + (int)rewind::Err; names = err_name (errors.cpp:8-31)
    import ctypes
    ref.L.ref_err_name.restype = ctypes.c_char_p
    for code in range(19):
        assert LIB.rw_status_name(code + 1).decode() == ref.L.ref_err_name(code).decode()


def test_invertibility_matches_reference(ref):
    for k in range(6):
        assert invertibility_check(k) == ref.L.ref_invertibility_check(k)


@pytest.mark.parametrize("field,value", [
    ("lr", 0.0), ("weight_decay", -1.0), ("momentum", 1.5), ("dampening", -0.1),
    ("beta1", 1.0), ("beta2", -0.5), ("eps", 0.0), (None, None)])
def test_validate_matches_reference(ref, field, value):
    h = OptimizerHyper(kind=2)
    if field:
        setattr(h, field, value)
    ref_st = ref.L.ref_validate(C.byref(ref.hyper(h)))
    ours = LIB.rw_hyper_validate(C.byref(h.to_c()))
    assert ours == ref_st


def test_lr_at_matches_reference(ref):
    h = OptimizerHyper(lr=0.1, lr_table=[(1, 0.1), (10, 0.05), (20, 0.01)])
    for t in (1, 5, 10, 11, 20, 1000):
        assert h.lr_at(t) == ref.lr_at(h, t)
    bad = OptimizerHyper(lr=0.1, lr_table=[(5, -1.0)])
    with pytest.raises(RwError) as e:
        bad.lr_at(6)
    assert e.value.name == "InvalidConfig"


def test_bubble_ratio_matches_reference(ref):
    for p in range(1, 17):
        for m in range(1, 17):
            a, b = C.c_int64(), C.c_int64()
            check(LIB.rw_bubble_ratio(p, m, C.byref(a), C.byref(b)))
            assert (a.value, b.value) == ref.bubble_ratio(p, m)
    with pytest.raises(RwError):
        check(LIB.rw_bubble_ratio(0, 4, C.byref(a), C.byref(b)))


def test_flat_layout_alignment():
    offs, total = flat_layout([1, 64, 65, 3])
    assert offs == [0, 64, 128, 256] and total == 320
    with pytest.raises(RwError):
        flat_layout([4, 0])


def test_state_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    g = (rw_group * 1)()
    g[0].offset, g[0].len = 0, 4
    buf = (C.c_float * 16)()
    st = LIB.rw_state_create(C.byref(h), 0, C.cast(buf, C.c_void_p), C.cast(buf, C.c_void_p),
                             None, None, None, 4, g, 1, 0)
    assert st == _lib.RW_CUDA_ERROR
    assert b"no CUDA device" in LIB.rw_last_error_message()


# ----------------------------- resolver (C++) vs the Python restatement
def _c_resolve(ranks, ready, kind=2, policy=0):
    """Run the two-phase all-reduce protocol in-process (MIN/MAX reductions)."""
    from oracle.oracle import resolve  # noqa: F401
    h = OptimizerHyper(kind=kind).to_c()
    tabs = []
    for r in ranks:
        g = (rw_group * len(r))()
        for i, (t, u) in enumerate(r):
            g[i].offset, g[i].len, g[i].t, g[i].updated = i * 64, 10, t, u
        tabs.append(g)
    loc = []
    for g, r in zip(tabs, ranks):
        s = rw_resolve_summary()
        check(LIB.rw_resolve_summarize(g, len(r), None, C.byref(h), 2**64 - 1, C.byref(s)))
        loc.append(s)
    lo, hi = min(s.t_min for s in loc), max(s.t_max for s in loc)
    glob = rw_resolve_summary()
    glob.t_min, glob.t_max = lo, hi
    for g, r, rd in zip(tabs, ranks, ready):
        s = rw_resolve_summary()
        arr = (C.c_uint8 * len(r))(*[1 if x else 0 for x in rd])
        check(LIB.rw_resolve_summarize(g, len(r), arr, C.byref(h), lo, C.byref(s)))
        for f in ("undo_elems", "redo_elems", "redo_blocked", "undo_blocked"):
            setattr(glob, f, max(getattr(glob, f), getattr(s, f)))
    out = []
    strat = None
    for g, r in zip(tabs, ranks):
        acts = (C.c_uint8 * len(r))()
        tgt, st = C.c_uint64(), C.c_int32()
        check(LIB.rw_resolve_plan(C.byref(glob), policy, g, len(r), acts, C.byref(tgt), C.byref(st)))
        out.append([["none", "undo", "redo"][a] for a in acts])
        strat = (_lib.STRATEGY_NAMES[st.value], tgt.value)
    return strat[0], strat[1], out


def test_resolver_matches_restatement_randomised():
    from oracle.oracle import resolve
    rng = random.Random(5)
    for trial in range(300):
        n_ranks = rng.randint(1, 4)
        n_groups = rng.randint(1, 8)
        base = rng.randint(0, 50)
        spread = rng.choice([1, 1, 1, 2])
        ranks = [[(base + rng.randint(0, spread), rng.randint(0, 1)) for _ in range(n_groups)]
                 for _ in range(n_ranks)]
        ready = [[rng.random() < 0.8 for _ in range(n_groups)] for _ in range(n_ranks)]
        kind = rng.choice([2, 5])  # Adam or AMSGrad (not invertible)
        policy = rng.choice([0, 1])
        ours = _c_resolve(ranks, ready, kind, policy)
        # restatement counts groups; C counts elements (all len 10) -> same order
        exp = resolve(ranks, ready, invertible=(kind == 2),
                      policy="min_cost" if policy else "undo")
        assert ours == exp, (ranks, ready, kind, policy)


# ----------------------------- planner (C++) vs restatement + brute force
def test_planner_spec_example_and_bruteforce():
    from oracle.oracle import brute_force_group_oracle, group_machines, plan_cost
    GB = 1e9
    res = planner.group_machines([1.0] * 4, [GB] * 3, GB, 100, 200 * GB)
    assert res.groups == [[0, 1], [2], [3]] and res.storage == 200 * GB
    rng = np.random.default_rng(11)
    gaps = []
    for trial in range(200):
        N = int(rng.integers(1, 9))
        R = list(rng.uniform(0.5, 2.0, N))
        M = list(rng.choice([0.0, 1.0, 2.0, 3.0], N - 1) * GB)
        T = float(rng.integers(1, 200))
        par = bool(rng.integers(0, 2))
        Mmax = float(rng.uniform(0, T * sum(M) + 1)) if N > 1 else 0.0
        ours = planner.group_machines(R, M, GB, T, Mmax, parallel=par)
        assert ours.storage <= Mmax + 1e-6                       # budget satisfied
        exp = group_machines(R, M, GB, T, Mmax, parallel=par)
        assert ours.groups == exp
        best = brute_force_group_oracle(R, M, GB, T, Mmax, parallel=par)
        b_rec = plan_cost(best, R, M, GB, T, N, par)[1]
        assert ours.recovery >= b_rec - 1e-12
        gaps.append(ours.recovery / b_rec)
        est = planner.recovery_time_estimate(R, M, GB, ours.groups, 50, parallel=par)
        assert est == pytest.approx(50 * plan_cost(ours.groups, R, M, GB, T, N, par)[1])
    assert min(gaps) >= 1.0 - 1e-12


def test_logging_worthwhile_matches_restatement():
    from oracle.oracle import logging_worthwhile
    for (b, bw, p, m, it) in [(1e9, 25e9, 8, 8, 1.0), (0.0, 25e9, 1, 4, 1.0), (1e9, 25e9, 1, 4, 1.0),
                              (1e12, 25e9, 4, 4, 1.0), (4 * 1024 * 128 * 2, 1e9, 4, 4, 0.01)]:
        ours = planner.logging_worthwhile(b, bw, p, m, it)
        exp = logging_worthwhile(b, bw, p, m, it)
        assert ours[0] == exp[0]
        assert ours[1] == pytest.approx(exp[1]) and ours[2] == pytest.approx(exp[2])
    # mb=4, hidden=1024, seq=128 -> 524,288 elements per boundary message
    assert planner.boundary_elems(4, 1024, 128) == 524288


def test_state_create_rejects_zero_extent_and_overflow():
    """shape_elements (tensor.cpp:52-56): a zero extent is InvalidShape; a group
    past the end of the state too -- both checked before any device work."""
    buf = (C.c_double * 64)()
    base = (C.addressof(buf) + 15) // 16 * 16
    out = C.c_void_p()
    for groups in ([(0, 4), (8, 0)], [(0, 4), (8, 100)]):
        arr = (rw_group * len(groups))()
        for i, (o, n) in enumerate(groups):
            arr[i].offset, arr[i].len = o, n
        st = LIB.rw_state_create(C.byref(out), 1, C.c_void_p(base), C.c_void_p(base), None, None, None, 32,
                                 arr, len(groups), 0)
        assert LIB.rw_status_name(st).decode() == "InvalidShape"


def test_resolver_empty_rank_is_identity():
    """A replacement with no state (n == 0) reports the identities of MIN / MAX
    (t_min = UINT64_MAX, t_max = 0), so a C++ host that all-reduces the raw
    summaries never drags the consensus to 0."""
    h = OptimizerHyper(kind=2).to_c()
    s = rw_resolve_summary()
    check(LIB.rw_resolve_summarize(None, 0, None, C.byref(h), 2**64 - 1, C.byref(s)))
    assert s.t_min == 2**64 - 1 and s.t_max == 0
    assert s.undo_elems == s.redo_elems == s.redo_blocked == 0
    # survivors at 10 / 11 plus an empty replacement -> the survivors' consensus
    assert _c_resolve([[(10, 0), (11, 1)], []], [[False, False], []])[:2] == ("Undo", 10)
