"""Pin the oracle before trusting it (CPU only).

1. The reference library (oracle/_ref, built from /root/reference) reproduces
   the SPEC known-answer vectors recorded in
   tests/golden/spec_vectors.json.
2. Our C restatement (oracle/restate.c) in fp64 equals the reference
   bit for bit on randomised blocks for every optimizer kind, step and undo.
3. The fp32 restatement is the fp64 one evaluated in float: checked to stay
   within the documented ulp tolerance of the fp64 reference.
"""
import math

import numpy as np
import pytest

from oracle.oracle import (ADAM, ADAMW, AMSGRAD, LAMB, SGD, SGDM, RefError, brute_force_group_oracle,
                           group_machines, parallel_assignment, plan_cost, resolve)

F = float.fromhex


def test_spec_vectors_reference(ref, golden):
    s = golden["spec"]
    assert [F(v) for v in s["sgd_step"]] == [1.8979999999999999]
    assert [F(v) for v in s["sgd_undo"]] == [2.0]
    assert s["double_undo"] == "NothingToUndo"
    assert [F(v) for v in s["sgdm_step_m"]] == [1.0]
    assert [F(v) for v in s["sgdm_step_x"]] == [0.9]
    assert s["sgdm_mu0_undo"] == "NonInvertibleHyper"
    assert s["amsgrad_require_invertible"] == "NotInvertible"
    assert s["amsgrad_undo"] == "NotInvertible"
    assert F(s["l2_norm_3_4"]) == 5.0
    assert s["bubble_4_4"] == [3, 7] and s["bubble_8_4"] == [7, 11]
    assert "P3 | .  .  .  F0 B0 F1 B1 F2 B2 F3 B3" in s["grid_4_4"]  # Fig 1a
    assert [F(v) for v in s["seeded_fill_2x2_7"]] == [
        -0.052143105428545056, 0.084315611201815799, 0.051316906045373471, 0.02008163517873536]
    assert s["crc32_123456789"] == 0xCBF43926
    # and the live reference still agrees with the committed fixture
    assert [v.hex() for v in ref.seeded_fill(4, 7)] == s["seeded_fill_2x2_7"]
    assert ref.crc32(b"123456789") == 0xCBF43926


def test_bubble_ratio_exhaustive(ref):
    # bubble_ratio equals the slot fraction for all p, m in [1,16]
    for p in range(1, 17):
        for m in range(1, 17):
            num, den = ref.bubble_ratio(p, m)
            sched = ref.schedule(p, m)
            slots = len(sched[0])
            bubbles = sum(1 for row in sched for k, _ in row if k == 2)
            assert slots == 2 * (m + p - 1)
            assert bubbles * den == num * p * slots
            assert num * (m + p - 1) == (p - 1) * den


HYPERS = {
    SGD: dict(kind=SGD, lr=0.05, weight_decay=0.01),
    SGDM: dict(kind=SGDM, lr=0.1, momentum=0.9, dampening=0.1, weight_decay=1e-4),
    ADAM: dict(kind=ADAM, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01),
    ADAMW: dict(kind=ADAMW, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01),
}


def _rand_state(rng, n, kind):
    x = rng.uniform(-1, 1, n)
    g = rng.uniform(-0.1, 0.1, n)
    m = rng.uniform(-0.05, 0.05, n) if kind != SGD else np.zeros(n)
    v = rng.uniform(0, 1e-3, n) if kind in (ADAM, ADAMW) else np.zeros(n)
    return x, g, m, v


@pytest.mark.parametrize("kind", [SGD, SGDM, ADAM, ADAMW])
def test_restatement_fp64_bitexact_vs_reference(ref, restate, kind):
    rng = np.random.default_rng(100 + kind)
    for trial in range(6):
        n = int(rng.integers(1, 3000))
        t0 = int(rng.integers(0, 100))
        h = dict(HYPERS[kind])
        h["lr_table"] = [(1, h["lr"]), (50, h["lr"] * 0.5)]
        x, g, m, v = _rand_state(rng, n, kind)
        b = ref.block(n)
        b.set(x=x, g=np.zeros(n), m=m, v=v, t=t0, updated=False)
        b.step(g, h)
        s1 = b.get()
        rx, rm, rv, _ = restate.step(kind, h, t0, x, g, m, v)
        assert s1["t"] == t0 + 1 and s1["updated"]
        assert np.array_equal(rx.view(np.uint64), s1["x"].view(np.uint64))
        assert np.array_equal(rm.view(np.uint64), s1["m"].view(np.uint64))
        assert np.array_equal(rv.view(np.uint64), s1["v"].view(np.uint64))
        assert np.array_equal(s1["g"], g)
        b.undo(h)
        s2 = b.get()
        ux, um, uv, _ = restate.undo(kind, h, t0 + 1, s1["x"], g, s1["m"], s1["v"])
        assert s2["t"] == t0 and not s2["updated"]
        assert np.array_equal(ux.view(np.uint64), s2["x"].view(np.uint64))
        assert np.array_equal(um.view(np.uint64), s2["m"].view(np.uint64))
        assert np.array_equal(uv.view(np.uint64), s2["v"].view(np.uint64))
        # SPEC:132 round trip <= 1e-9 relative (not bit-identical, Appendix B)
        for a, b0 in ((s2["x"], x), (s2["m"], m), (s2["v"], v)):
            den = np.maximum(np.abs(b0), 1e-300)
            assert np.all(np.abs(a - b0) <= 1e-9 * np.maximum(den, np.abs(a)) + 1e-300)


def test_restatement_amsgrad_and_lamb_fp64(ref, restate):
    rng = np.random.default_rng(7)
    n = 513
    x, g, m, v = _rand_state(rng, n, ADAM)
    h = dict(kind=AMSGRAD, lr=1e-3, weight_decay=0.01)
    b = ref.block(n)
    b.set(x=x, g=np.zeros(n), m=m, v=v, t=4)
    b.step(g, h)
    s1 = b.get()
    rx, rm, rv, rvm, _ = restate.step_amsgrad(h, 4, x, g, m, v, np.zeros(n))
    assert np.array_equal(rx, s1["x"]) and np.array_equal(rm, s1["m"]) and np.array_equal(rv, s1["v"])
    # LAMB: step saves the trust ratio, undo consumes it (optim.cpp:195-242)
    import ctypes as C
    from oracle.oracle import _dptr
    hl = dict(kind=LAMB, lr=1e-3, weight_decay=0.01)
    b = ref.block(n)
    b.set(x=x, g=np.zeros(n), m=m, v=v, t=2)
    b.step(g, hl)
    s1 = b.get()
    trust = b.saved_scalars()[-1]
    s = restate.scalars(hl, 2, False)
    xx, mm, vv = x.copy(), m.copy(), v.copy()
    tr = C.c_double()
    restate.L.oracle_step_lamb_f64(C.byref(s), _dptr(xx), _dptr(g), _dptr(mm), _dptr(vv), n, C.byref(tr))
    assert tr.value == trust
    assert np.array_equal(xx, s1["x"]) and np.array_equal(mm, s1["m"])
    b.undo(hl)
    s2 = b.get()
    su = restate.scalars(hl, 3, True)
    restate.L.oracle_undo_lamb_f64(C.byref(su), trust, _dptr(xx), _dptr(g), _dptr(mm), _dptr(vv), n)
    assert np.array_equal(xx, s2["x"]) and np.array_equal(mm, s2["m"]) and np.array_equal(vv, s2["v"])


@pytest.mark.parametrize("kind", [SGD, SGDM, ADAM, ADAMW])
def test_restatement_fp32_close_to_reference(ref, restate, kind):
    """fp32 restatement vs the fp64 reference on the same (fp32-representable)
    inputs: |d| <= 4 ulp_fp32(max |operand|) per output."""
    rng = np.random.default_rng(200 + kind)
    n = 4096
    x, g, m, v = (a.astype(np.float32).astype(np.float64) for a in _rand_state(rng, n, kind))
    h = HYPERS[kind]
    rx64, rm64, rv64, _ = restate.step(kind, h, 5, x, g, m, v)
    rx32, rm32, rv32, _ = restate.step(kind, h, 5, x, g, m, v, dtype=np.float32)

    def ulp(a):
        return np.spacing(np.abs(a).astype(np.float32)).astype(np.float64)

    assert np.all(np.abs(rx32 - rx64) <= 4 * ulp(np.maximum(np.abs(x), np.abs(rx64))) + 1e-30)
    if kind != SGD:
        bound = np.maximum.reduce([np.abs(m), np.abs(g), np.abs(rm64)])
        assert np.all(np.abs(rm32 - rm64) <= 4 * ulp(bound) + 1e-30)


def test_seeded_fill_and_seeds_restated(ref, restate):
    for seed in (0, 1, 7, 2302, 2**63 + 5):
        a = ref.seeded_fill(1000, seed)
        b = restate.seeded_fill(1000, seed)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    for parts in ([], [0], [0, 1], [3, 4, 5], [1, 2, 3, 4]):
        assert ref.derive_seed(2302, parts) == restate.derive_seed(2302, parts)


def test_ordered_sum_restated(ref, restate):
    rng = np.random.default_rng(3)
    arrs = [rng.standard_normal(777) * 10.0 ** rng.integers(-3, 3) for _ in range(9)]
    a = ref.ordered_sum(arrs)
    b = restate.ordered_sum(arrs)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    with pytest.raises(RefError) as e:
        ref.ordered_sum([])
    assert e.value.name == "EmptyInput"
    with pytest.raises(RefError) as e:
        ref.ordered_sum([np.zeros(3), np.zeros(4)])
    assert e.value.name == "ShapeMismatch"


# ------------------------------------------ SPEC-only restatements
def test_resolver_restatement_examples():
    # SPEC:481-483 consensus = min
    assert resolve([[(150, 0)], [(150, 0)], [(151, 0)]])[1] == 150
    # Fig 5: only layer N-1 updated on the survivor -> undo exactly that one
    strat, target, acts = resolve([[(10, 0), (10, 0), (11, 1)]])
    assert strat == "Undo" and target == 10 and acts == [["none", "none", "undo"]]
    # no flags -> no-op
    assert resolve([[(10, 0), (10, 0)]])[0] == "None"
    # AMSGrad (not invertible), no gradients ready -> global rollback
    assert resolve([[(10, 0), (11, 1)]], invertible=False)[0] == "GlobalRollback"
    # two steps apart -> rollback
    assert resolve([[(10, 0), (12, 1)]])[0] == "GlobalRollback"
    # redo when cheaper and every lagging group holds its gradient
    strat, target, acts = resolve([[(10, 0), (11, 1), (11, 1)]], [[True, False, False]],
                                  policy="min_cost")
    assert strat == "Redo" and target == 11 and acts == [["redo", "none", "none"]]


def test_planner_restatement_spec_example():
    # N=4, R=1s, M=1GB, B=1GB/s, T=100, M_max=200GB -> [[0,1],[2],[3]]
    GB = 1e9
    R, M = [1.0] * 4, [GB] * 3
    g = group_machines(R, M, GB, 100, 200 * GB)
    assert g == [[0, 1], [2], [3]]
    assert plan_cost(g, R, M, GB, 100, 4, False)[0] == 200 * GB
    assert group_machines(R, M, GB, 100, 1e30) == [[0], [1], [2], [3]]
    assert group_machines(R, M, GB, 100, 0.0) == [[0, 1, 2, 3]]
    ob = brute_force_group_oracle(R, M, GB, 100, 200 * GB)
    assert math.isclose(plan_cost(ob, R, M, GB, 100, 4, False)[1],
                        plan_cost(g, R, M, GB, 100, 4, False)[1])
    assert parallel_assignment(4, 2) == [[0, 2], [1, 3]]  # Fig 6


def test_subpipeline_1f1b_order_matches_reference_schedule(ref):
    """The per-worker order the stage-per-GPU sub-pipeline executes
    (subpipeline.one_f_one_b) is exactly the non-bubble slot sequence of the
    reference's build_1f1b_schedule (schedule.cpp:25-84) for every worker,
    exhaustively for p, m <= 16."""
    from paper_2302_06173_b200.subpipeline import one_f_one_b
    for p in range(1, 17):
        for m in range(1, 17):
            sch = ref.schedule(p, m)
            for w in range(p):
                got = [("F" if k == 0 else "B", mb) for k, mb in sch[w] if k != 2]
                assert got == one_f_one_b(p, m, w), (p, m, w)
