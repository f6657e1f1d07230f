"""LAMB on the device against the restatement of
step_lamb / undo_lamb (optim.cpp:195-242; oracle/restate.c, pinned bit-exact
to the reference in test_oracle.py).

Bars:
  * m, v after the step: bit-exact (elementwise, same op order);
  * trust ratio: the device sums ||x||^2 and ||update||^2 in fp64 with a fixed
    tree order, the reference left to right, so the ratio differs in the last
    bits: |rel| <= 2 n 2^-53 (the n*u bound of a sequential sum, per group);
  * x after the step: bit-exact GIVEN the device's trust ratio (recomputed here
    in numpy with the reference's op order), and within the trust tolerance of
    the restatement;
  * undo: bit-exact vs undo_lamb with the same saved ratio; the saved-scalar
    stack behaves like ParamBlock::saved_scalars (push on step, pop on undo,
    NothingToUndo when empty).
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle.oracle import _dptr
from paper_2302_06173_b200 import LAMB, DeviceState, OptimizerHyper, RwError
from paper_2302_06173_b200._lib import LIB, check

pytestmark = pytest.mark.gpu

H = OptimizerHyper(kind=LAMB, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=0.01)
SIZES = [1000, 70001, 5, 4096]


def _fill(st, rng, t0):
    for i, n in enumerate(st.sizes):
        st.view("x", i).copy_(torch.from_numpy(rng.standard_normal(n)))
        st.view("m", i).copy_(torch.from_numpy(rng.standard_normal(n) * 1e-2))
        st.view("v", i).copy_(torch.from_numpy(np.abs(rng.standard_normal(n)) * 1e-4))
    st.write_markers([(t0, 0)] * st.num_groups)


def _np(st, which, i):
    return st.view(which, i).cpu().numpy().copy()


def test_lamb_step_undo_fp64(restate):
    rng = np.random.default_rng(11)
    t0 = 3
    st = DeviceState(SIZES, dtype=torch.float64, kind=LAMB)
    _fill(st, rng, t0)
    grad = torch.zeros(st.total, dtype=torch.float64, device="cuda")
    grad.copy_(torch.from_numpy(rng.standard_normal(st.total)))
    before = {w: [_np(st, w, i) for i in range(st.num_groups)] for w in ("x", "m", "v")}
    st.step(H, grad=grad)  # reverse layer order
    st.check_finite()
    assert st.markers() == [(t0 + 1, 1)] * st.num_groups
    s = restate.scalars(H, t0, False)
    for i, n in enumerate(SIZES):
        g = grad[st.offsets[i]:st.offsets[i] + n].cpu().numpy()
        x0, m0, v0 = (before[w][i].copy() for w in ("x", "m", "v"))
        xx, mm, vv = x0.copy(), m0.copy(), v0.copy()
        tr = C.c_double()
        restate.L.oracle_step_lamb_f64(C.byref(s), _dptr(xx), _dptr(g), _dptr(mm), _dptr(vv), n, C.byref(tr))
        assert np.array_equal(_np(st, "m", i), mm) and np.array_equal(_np(st, "v", i), vv)
        assert np.array_equal(_np(st, "g", i), g)  # block.g = grad (optim.cpp:271)
        saved = st.saved_scalars(i)
        assert len(saved) == 1
        trust = saved[0]
        assert abs(trust - tr.value) <= 2 * n * 2.0**-53 * abs(tr.value)
        # pass 2 bit-exact given the device trust, reference op order
        mhat, vhat = mm / s.c1, vv / s.c2
        upd = mhat / (np.sqrt(vhat) + s.eps) + s.wd * x0
        x_exp = x0 - (s.eta * trust) * upd
        assert np.array_equal(_np(st, "x", i), x_exp)
        assert np.allclose(_np(st, "x", i), xx, rtol=0, atol=4 * n * 2.0**-53 * np.max(np.abs(x0)))
    # undo: bit-exact vs undo_lamb with the same saved ratio
    su = restate.scalars(H, t0 + 1, True)
    exp = {}
    for i, n in enumerate(SIZES):
        xx, mm, vv = (_np(st, w, i) for w in ("x", "m", "v"))
        g = _np(st, "g", i)
        restate.L.oracle_undo_lamb_f64(C.byref(su), st.saved_scalars(i)[0], _dptr(xx), _dptr(g), _dptr(mm),
                                       _dptr(vv), n)
        exp[i] = (xx, mm, vv)
    st.undo(H)
    st.check_finite()
    assert st.markers() == [(t0, 0)] * st.num_groups
    for i in range(len(SIZES)):
        assert np.array_equal(_np(st, "x", i), exp[i][0])
        assert np.array_equal(_np(st, "m", i), exp[i][1])
        assert np.array_equal(_np(st, "v", i), exp[i][2])
        assert st.saved_scalars(i) == []
        # the round trip lands within rounding of the pre-step state
        assert np.allclose(_np(st, "x", i), before["x"][i], rtol=1e-12, atol=1e-14)


def test_lamb_saved_scalar_stack_and_guards():
    rng = np.random.default_rng(5)
    st = DeviceState([300, 77], dtype=torch.float64, kind=LAMB)
    _fill(st, rng, 0)
    g1 = torch.from_numpy(rng.standard_normal(st.total)).cuda()
    g2 = torch.from_numpy(rng.standard_normal(st.total)).cuda()
    st.step(H, grad=g1)
    st.clear_updated()
    st.step(H, grad=g2)
    assert [len(st.saved_scalars(i)) for i in range(2)] == [2, 2]
    t1 = [st.saved_scalars(i) for i in range(2)]
    # pop in order: undo uses the top ratio (the second step's)
    st.undo(H)
    assert [st.saved_scalars(i) for i in range(2)] == [t[:1] for t in t1]
    # undo of the first step: g must hold the first step's gradient again
    st.g.copy_(g1)
    st.write_markers([(1, 1)] * 2)
    st.undo(H)
    assert [st.saved_scalars(i) for i in range(2)] == [[], []]
    assert st.markers() == [(0, 0), (0, 0)]
    # NothingToUndo: no saved ratio even though the marker is armed
    st.write_markers([(1, 1)] * 2)
    with pytest.raises(RwError) as e:
        st.undo(H, [0])
    assert "saved trust" in str(e.value)
    # set/read round trip (replication of the stack)
    st.set_saved_scalars(1, [0.5, 0.25])
    assert st.saved_scalars(1) == [0.5, 0.25]
    # NonInvertibleHyper: beta1 == 0
    hb = OptimizerHyper(kind=LAMB, lr=1e-3, beta1=0.0, beta2=0.999, eps=1e-6, weight_decay=0.01)
    with pytest.raises(RwError) as e:
        st.undo(hb, [1])
    assert "beta1*beta2" in str(e.value)
    # trust*lr*weight_decay == 1
    st.set_saved_scalars(1, [1.0])
    hw = OptimizerHyper(kind=LAMB, lr=0.5, beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=2.0)
    with pytest.raises(RwError) as e:
        st.undo(hw, [1])
    assert "trust*lr*weight_decay" in str(e.value)


def test_lamb_crash_mid_update_and_resolve():
    """MidUpdate(k) with LAMB: the resolver's undo plan rolls back exactly the
    stepped groups using their saved ratios (single process, no peers)."""
    from paper_2302_06173_b200.recovery import apply_resolution, resolve
    rng = np.random.default_rng(9)
    st = DeviceState([128, 256, 512, 1024], dtype=torch.float64, kind=LAMB)
    _fill(st, rng, 5)
    x0 = st.x.clone()
    grad = torch.from_numpy(rng.standard_normal(st.total)).cuda()
    st.step(H, grad=grad, stop_after=2)  # groups 3, 2 stepped
    mk = st.markers()
    assert mk == [(5, 0), (5, 0), (6, 1), (6, 1)]
    plan = resolve(mk, H, lens=st.sizes)
    assert plan.strategy == "Undo" and sorted(plan.undo_ids) == [2, 3]
    apply_resolution(st, H, plan)
    assert st.markers() == [(5, 0)] * 4
    assert torch.allclose(st.x, x0, rtol=1e-12, atol=1e-14)


def test_lamb_fp32_close_to_fp64(restate):
    rng = np.random.default_rng(3)
    n = 5000
    st = DeviceState([n], dtype=torch.float32, kind=LAMB)
    x0 = rng.standard_normal(n).astype(np.float32)
    m0 = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    v0 = (np.abs(rng.standard_normal(n)) * 1e-4).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    for w, a in (("x", x0), ("m", m0), ("v", v0)):
        st.view(w, 0).copy_(torch.from_numpy(a))
    st.write_markers([(2, 0)])
    gd = torch.zeros(st.total, dtype=torch.float32, device="cuda")
    gd[:n] = torch.from_numpy(g)
    st.step(H, grad=gd)
    s = restate.scalars(H, 2, False)
    xx, mm, vv = x0.astype(np.float64), m0.astype(np.float64), v0.astype(np.float64)
    tr = C.c_double()
    restate.L.oracle_step_lamb_f64(C.byref(s), _dptr(xx), _dptr(g.astype(np.float64)), _dptr(mm), _dptr(vv), n,
                                   C.byref(tr))
    assert abs(st.saved_scalars(0)[0] - tr.value) <= 1e-5 * tr.value
    assert np.allclose(_np(st, "x", 0), xx, rtol=1e-5, atol=1e-6)
    st.undo(H)
    assert np.allclose(_np(st, "x", 0), x0, rtol=1e-5, atol=1e-6)


def test_host_block_lamb_matches_restatement(restate):
    """rw_host_block_lamb_step/undo: one reference ParamBlock in host memory."""
    rng = np.random.default_rng(21)
    n = 777
    x = rng.standard_normal(n)
    m = rng.standard_normal(n) * 1e-2
    v = np.abs(rng.standard_normal(n)) * 1e-4
    grad = rng.standard_normal(n)
    g = np.zeros(n)
    t, upd = C.c_uint64(4), C.c_uint32(0)
    trust = C.c_double()
    xs, ms, vs = x.copy(), m.copy(), v.copy()
    h = H.to_c()
    check(LIB.rw_host_block_lamb_step(1, _dptr(xs), _dptr(g), _dptr(ms), _dptr(vs), n, C.byref(t), C.byref(upd),
                                      _dptr(grad), C.byref(h), C.byref(trust)))
    assert (t.value, upd.value) == (5, 1)
    s = restate.scalars(H, 4, False)
    xx, mm, vv = x.copy(), m.copy(), v.copy()
    tr = C.c_double()
    restate.L.oracle_step_lamb_f64(C.byref(s), _dptr(xx), _dptr(grad), _dptr(mm), _dptr(vv), n, C.byref(tr))
    assert np.array_equal(ms, mm) and np.array_equal(vs, vv) and np.array_equal(g, grad)
    # the host-block path forms the norms left to right (RW_STATE_LAMB_SEQUENTIAL_NORMS):
    # the trust ratio and x are the reference's bits
    assert trust.value == tr.value
    assert np.array_equal(xs, xx)
    su = restate.scalars(H, 5, True)
    ex, em, ev = xs.copy(), ms.copy(), vs.copy()
    restate.L.oracle_undo_lamb_f64(C.byref(su), trust.value, _dptr(ex), _dptr(g), _dptr(em), _dptr(ev), n)
    check(LIB.rw_host_block_lamb_undo(1, _dptr(xs), _dptr(g), _dptr(ms), _dptr(vs), n, C.byref(t), C.byref(upd),
                                      C.byref(h), 1, trust.value))
    assert (t.value, upd.value) == (4, 0)
    assert np.array_equal(xs, ex) and np.array_equal(ms, em) and np.array_equal(vs, ev)
    # no saved ratio -> NothingToUndo, nothing touched
    upd.value = 1
    st = LIB.rw_host_block_lamb_undo(1, _dptr(xs), _dptr(g), _dptr(ms), _dptr(vs), n, C.byref(t), C.byref(upd),
                                     C.byref(h), 0, 0.0)
    assert st == 7  # RW_NOTHING_TO_UNDO
    assert (t.value, upd.value) == (4, 1)
