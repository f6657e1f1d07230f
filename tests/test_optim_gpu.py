"""GPU parity of the fused step/undo kernels (through the C ABI).

Bars (north_star):
  * fp64 kernels: bit-exact vs the reference library (golden fixtures from
    oracle/_ref and the live fp64 restatement, itself pinned bit-exact to _ref);
  * fp32 kernels: bit-exact vs the fp32 restatement (reference operation order
    in float, no FMA contraction);
  * markers, guards and error codes identical to optimizer_step/undo.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import Restate
from paper_2302_06173_b200 import (ADAM, ADAMW, AMSGRAD, SGD, SGDM, DeviceState, OptimizerHyper,
                                   RwError, ordered_sum, seeded_fill_)

pytestmark = pytest.mark.gpu

F = float.fromhex
HYP = {
    SGD: OptimizerHyper(kind=SGD, lr=0.05, weight_decay=0.01),
    SGDM: OptimizerHyper(kind=SGDM, lr=0.1, momentum=0.9, dampening=0.1, weight_decay=1e-4),
    ADAM: OptimizerHyper(kind=ADAM, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01),
    ADAMW: OptimizerHyper(kind=ADAMW, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01),
}
NAMES = {"sgd": SGD, "sgdm": SGDM, "adam": ADAM, "adamw": ADAMW}


def _bits(a):
    a = np.asarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def _load(st: DeviceState, i, x, g, m, v):
    dt = st.dtype
    st.view("x", i).copy_(torch.as_tensor(x, dtype=dt))
    st.view("g", i).copy_(torch.as_tensor(g, dtype=dt))
    if st.m is not None:
        st.view("m", i).copy_(torch.as_tensor(m, dtype=dt))
    if st.v is not None:
        st.view("v", i).copy_(torch.as_tensor(v, dtype=dt))


def _get(st, which, i):
    return st.view(which, i).cpu().numpy()


@pytest.mark.parametrize("name", ["sgd", "sgdm", "adam", "adamw"])
def test_fp64_bitexact_vs_reference_golden(golden, name):
    blk = golden["blocks"][name]
    kind = NAMES[name]
    h = OptimizerHyper(**{k: v for k, v in blk["hyper"].items()})
    x0, g, m0, v0 = ([F(s) for s in blk[k]] for k in ("x0", "g", "m0", "v0"))
    n = len(x0)
    st = DeviceState([n], dtype=torch.float64, kind=kind)
    _load(st, 0, x0, np.zeros(n), m0, v0)
    st.write_markers([(blk["t0"], 0)])
    grad = torch.zeros(st.total, dtype=torch.float64, device="cuda")
    grad[:n] = torch.tensor(g, dtype=torch.float64)
    st.step(h, [0], grad=grad)
    st.check_finite()
    assert st.markers() == [(blk["t0"] + 1, 1)]
    assert np.array_equal(_bits(_get(st, "x", 0)), _bits([F(s) for s in blk["step"]["x"]]))
    assert np.array_equal(_get(st, "g", 0), np.array(g))  # block.g = grad (optim.cpp:271)
    if kind != SGD:
        assert np.array_equal(_bits(_get(st, "m", 0)), _bits([F(s) for s in blk["step"]["m"]]))
    if kind in (ADAM, ADAMW):
        assert np.array_equal(_bits(_get(st, "v", 0)), _bits([F(s) for s in blk["step"]["v"]]))
    st.undo(h, [0])
    st.check_finite()
    assert st.markers() == [(blk["t0"], 0)]
    assert np.array_equal(_bits(_get(st, "x", 0)), _bits([F(s) for s in blk["undo"]["x"]]))
    if kind != SGD:
        assert np.array_equal(_bits(_get(st, "m", 0)), _bits([F(s) for s in blk["undo"]["m"]]))
    if kind in (ADAM, ADAMW):
        assert np.array_equal(_bits(_get(st, "v", 0)), _bits([F(s) for s in blk["undo"]["v"]]))


def _random_groups(rng, kind, sizes, dtype):
    out = []
    for n in sizes:
        x = rng.uniform(-1, 1, n)
        g = rng.uniform(-0.1, 0.1, n)
        m = rng.uniform(-0.05, 0.05, n) if kind != SGD else np.zeros(n)
        v = rng.uniform(0, 1e-3, n) if kind in (ADAM, ADAMW, AMSGRAD) else np.zeros(n)
        out.append(tuple(a.astype(dtype) for a in (x, g, m, v)))
    return out


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("kind", [SGD, SGDM, ADAM, ADAMW])
def test_multigroup_bitexact_vs_restatement(restate: Restate, kind, dtype):
    """Ragged groups (sizes not multiples of the vector width or chunk), each at
    its own t (distinct scalar sets in one launch), stepped in update order and
    then undone — compared bit for bit with the restatement."""
    rng = np.random.default_rng(kind * 10 + (dtype == np.float64))
    sizes = [1, 3, 7, 64, 100, 1023, 4097, 8191, 8193, 20000, 70001]
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    st = DeviceState(sizes, dtype=tdt, kind=kind)
    data = _random_groups(rng, kind, sizes, dtype)
    t0 = [int(rng.integers(0, 30)) for _ in sizes]
    for i, (x, g, m, v) in enumerate(data):
        _load(st, i, x, np.zeros_like(g), m, v)
    st.write_markers([(t, 0) for t in t0])
    grad = torch.zeros(st.total, dtype=tdt, device="cuda")
    for i, (x, g, m, v) in enumerate(data):
        grad[st.offsets[i]:st.offsets[i] + sizes[i]] = torch.as_tensor(g)
    h = HYP[kind]
    st.step(h, grad=grad)
    st.check_finite()
    assert st.markers() == [(t + 1, 1) for t in t0]
    stepped = []
    for i, (x, g, m, v) in enumerate(data):
        rx, rm, rv, _ = restate.step(kind, h, t0[i], x, g, m, v, dtype=dtype)
        assert np.array_equal(_bits(_get(st, "x", i)), _bits(rx)), (i, sizes[i])
        if kind != SGD:
            assert np.array_equal(_bits(_get(st, "m", i)), _bits(rm)), i
        if kind in (ADAM, ADAMW):
            assert np.array_equal(_bits(_get(st, "v", i)), _bits(rv)), i
        stepped.append((rx, g, rm, rv))
    st.undo(h)
    st.check_finite()
    assert st.markers() == [(t, 0) for t in t0]
    for i, (rx, g, rm, rv) in enumerate(stepped):
        ux, um, uv, _ = restate.undo(kind, h, t0[i] + 1, rx, g, rm, rv, dtype=dtype)
        assert np.array_equal(_bits(_get(st, "x", i)), _bits(ux)), i
        if kind != SGD:
            assert np.array_equal(_bits(_get(st, "m", i)), _bits(um)), i
        if kind in (ADAM, ADAMW):
            assert np.array_equal(_bits(_get(st, "v", i)), _bits(uv)), i


def test_many_groups_beyond_the_presized_slots(restate: Restate):
    """5,000 ragged groups at 40 distinct t: more work items than a launch slot
    is pre-sized for at state creation (4,096) and far beyond the inline
    parameter path (128 items / 16 scalar sets), so the slot grows inside the
    call; Adam step then undo of every group, bit for bit vs the restatement."""
    rng = np.random.default_rng(5000)
    sizes = [int(n) for n in rng.integers(1, 300, 5000)]
    st = DeviceState(sizes, dtype=torch.float32, kind=ADAM)
    data = _random_groups(rng, ADAM, sizes, np.float32)
    t0 = [int(rng.integers(0, 40)) for _ in sizes]
    flat = {k: np.zeros(st.total, np.float32) for k in "xgmv"}
    for i, grp in enumerate(data):  # one host image per buffer, one copy each
        o = st.offsets[i]
        for k, a in zip("xgmv", grp):
            flat[k][o:o + sizes[i]] = a
    for k in "xgmv":
        getattr(st, k).copy_(torch.from_numpy(flat[k]))
    st.write_markers([(t, 0) for t in t0])
    h = HYP[ADAM]
    st.step(h)
    st.undo(h)
    st.check_finite()
    assert st.markers() == [(t, 0) for t in t0]
    out = {k: getattr(st, k).cpu().numpy() for k in "xmv"}
    for i in range(0, len(sizes), 7):  # a deterministic sample of the groups
        x, g, m, v = data[i]
        rx, rm, rv, _ = restate.step(ADAM, h, t0[i], x, g, m, v, dtype=np.float32)
        ux, um, uv, _ = restate.undo(ADAM, h, t0[i] + 1, rx, g, rm, rv, dtype=np.float32)
        o, n = st.offsets[i], sizes[i]
        assert np.array_equal(_bits(out["x"][o:o + n]), _bits(ux)), i
        assert np.array_equal(_bits(out["m"][o:o + n]), _bits(um)), i
        assert np.array_equal(_bits(out["v"][o:o + n]), _bits(uv)), i


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_amsgrad_step_bitexact(restate, dtype):
    rng = np.random.default_rng(9)
    sizes = [5, 4099]
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    st = DeviceState(sizes, dtype=tdt, kind=AMSGRAD)
    h = OptimizerHyper(kind=AMSGRAD, lr=1e-3, weight_decay=0.01)
    data = _random_groups(rng, AMSGRAD, sizes, dtype)
    vmax0 = [rng.uniform(0, 1e-3, n).astype(dtype) for n in sizes]
    for i, (x, g, m, v) in enumerate(data):
        _load(st, i, x, g, m, v)
        st.view("vmax", i).copy_(torch.as_tensor(vmax0[i]))
    st.step(h)
    for i, (x, g, m, v) in enumerate(data):
        rx, rm, rv, rvm, _ = restate.step_amsgrad(h, 0, x, g, m, v, vmax0[i], dtype=dtype)
        assert np.array_equal(_bits(_get(st, "x", i)), _bits(rx))
        assert np.array_equal(_bits(_get(st, "vmax", i)), _bits(rvm))
    with pytest.raises(RwError) as e:
        st.undo(h)
    assert e.value.name == "NotInvertible"


def test_guards_match_reference_order():
    st = DeviceState([10, 10], kind=ADAM)
    h = HYP[ADAM]
    with pytest.raises(RwError) as e:
        st.undo(h, [0])
    assert e.value.name == "NothingToUndo"
    st.step(h, [1])
    with pytest.raises(RwError) as e:
        st.step(h, [0, 1])                       # group 1 already stepped
    assert e.value.name == "AlreadyUpdated"
    assert st.markers() == [(0, 0), (1, 1)]      # nothing launched for group 0
    with pytest.raises(RwError) as e:
        st.step(OptimizerHyper(kind=AMSGRAD, require_invertible=True), [0])
    assert e.value.name == "NotInvertible"
    with pytest.raises(RwError) as e:
        st.undo(OptimizerHyper(kind=ADAM, beta1=0.0), [1])
    assert e.value.name == "NonInvertibleHyper"
    with pytest.raises(RwError) as e:
        st.undo(OptimizerHyper(kind=ADAM, lr=0.1, lr_table=[(1, -1.0)]), [1])
    assert e.value.name == "InvalidConfig"
    st2 = DeviceState([4], kind=SGDM)
    st2.step(OptimizerHyper(kind=SGDM, momentum=0.0), [0])
    with pytest.raises(RwError) as e:
        st2.undo(OptimizerHyper(kind=SGDM, momentum=0.0), [0])
    assert e.value.name == "NonInvertibleHyper"
    st3 = DeviceState([4], kind=SGD)
    st3.step(OptimizerHyper(kind=SGD, lr=1.0, weight_decay=1.0), [0])
    with pytest.raises(RwError) as e:
        st3.undo(OptimizerHyper(kind=SGD, lr=1.0, weight_decay=1.0), [0])
    assert e.value.name == "NonInvertibleHyper"


def test_numerical_error_after_mutation():
    st = DeviceState([100, 100], kind=ADAM)
    st.g.fill_(0.01)
    st.g[st.offsets[1] + 7] = float("inf")
    st.step(HYP[ADAM])
    with pytest.raises(RwError) as e:
        st.check_finite()
    assert e.value.name == "NumericalError"
    # like the reference, the mutation happened and t/updated advanced
    assert st.markers() == [(1, 1), (1, 1)]
    assert not torch.isfinite(st.view("x", 1)).all()
    st.check_finite()  # flag consumed


def test_crash_injection_markers():
    """MidUpdate(k): after k groups in update order (reverse
    layer order) exactly those groups carry updated=1 and t+1."""
    G = 12
    st = DeviceState([3000 + 17 * i for i in range(G)], kind=SGDM)
    seeded_fill_(st.x, 11)
    h = HYP[SGDM]
    for k in (0, 1, 5, G):
        st.write_markers([(4, 0)] * G)
        st.step(h, stop_after=k)
        mk = st.markers()
        order = st.update_order()
        for pos, gi in enumerate(order):
            assert mk[gi] == ((5, 1) if pos < k else (4, 0)), (k, gi)


def test_seeded_fill_bit_identical_to_host(restate):
    for dt, npdt in ((torch.float64, np.float64), (torch.float32, np.float32)):
        out = torch.empty(100003, dtype=dt, device="cuda")
        seeded_fill_(out, 2302)
        host = restate.seeded_fill(100003, 2302, dtype=npdt)
        assert np.array_equal(_bits(out.cpu().numpy()), _bits(host))
    # counter offset = the same stream continued
    out = torch.empty(1000, dtype=torch.float64, device="cuda")
    seeded_fill_(out, 7, offset=500)
    assert np.array_equal(out.cpu().numpy(), restate.seeded_fill(1500, 7)[500:])


@pytest.mark.parametrize("count", [1, 2, 9, 70])
def test_ordered_sum_bit_identical(restate, count):
    rng = np.random.default_rng(count)
    for dt, npdt in ((torch.float64, np.float64), (torch.float32, np.float32)):
        arrs = [(rng.standard_normal(5001) * 10.0 ** rng.integers(-4, 4)).astype(npdt)
                for _ in range(count)]
        out = ordered_sum([torch.as_tensor(a, device="cuda") for a in arrs])
        assert np.array_equal(_bits(out.cpu().numpy()), _bits(restate.ordered_sum(arrs, dtype=npdt)))


def test_large_state_roundtrip_sampled(restate):
    """At a large size: step + undo in one launch each over 64 groups; check
    bitwise against the restatement on a random sample of elements (the ops are
    elementwise, so sampling is exact) and the SPEC:132 round-trip property."""
    sizes = [1_000_003 + 4099 * i for i in range(64)]
    st = DeviceState(sizes, kind=ADAM)
    seeded_fill_(st.x, 1)
    seeded_fill_(st.m, 2)
    st.m.mul_(0.01)
    seeded_fill_(st.v, 3)
    st.v.abs_().mul_(1e-4)
    grad = torch.empty_like(st.x)
    seeded_fill_(grad, 4)
    x0, m0, v0 = st.x.clone(), st.m.clone(), st.v.clone()
    st.write_markers([(7, 0)] * len(sizes))
    h = HYP[ADAM]
    st.step(h, grad=grad)
    xs = st.x.clone()
    gen = torch.Generator(device="cuda").manual_seed(0)
    gi = torch.randint(0, len(sizes), (200_000,), device="cuda", generator=gen)
    offs = torch.tensor(st.offsets, device="cuda")[gi]
    lens = torch.tensor(sizes, device="cuda")[gi]
    idx = offs + (torch.rand(200_000, device="cuda", generator=gen) * lens).long().clamp_max(lens - 1)
    rx, rm, rv, _ = restate.step(ADAM, h, 7, x0[idx].cpu().numpy(), grad[idx].cpu().numpy(),
                                 m0[idx].cpu().numpy(), v0[idx].cpu().numpy(), dtype=np.float32)
    assert np.array_equal(_bits(st.x[idx].cpu().numpy()), _bits(rx))
    assert np.array_equal(_bits(st.v[idx].cpu().numpy()), _bits(rv))
    st.undo(h)
    st.check_finite()
    ux, um, uv, _ = restate.undo(ADAM, h, 8, rx, grad[idx].cpu().numpy(), rm, rv, dtype=np.float32)
    assert np.array_equal(_bits(st.x[idx].cpu().numpy()), _bits(ux))
    assert np.array_equal(_bits(st.m[idx].cpu().numpy()), _bits(um))
    # fp32 round trip: x within 1 ulp of max(|x_t|, |x_t+1|)
    sp = torch.maximum(x0.abs(), xs.abs())
    assert ((st.x - x0).abs() <= 2 * torch.finfo(torch.float32).eps * sp + 1e-30).all()


@pytest.mark.parametrize("ids", [[5, 3, 1, 0], [3, 1]])
@pytest.mark.parametrize("kind,dtype", [(ADAM, torch.float32), (SGDM, torch.float32), (ADAM, torch.float64),
                                         ("lamb", torch.float32)])
def test_undo_from_host_pipelined_equals_device_undo(kind, dtype, ids):
    """rw_optimizer_undo_host (H2D | undo | D2H pipelined per slice through a
    three-slice device ring) gives the same bits and markers as the
    device-resident undo, for many small slices, on a host-resident state
    (rw_state_create_host: no device copy of x, g, m, v); groups not undone
    reach `out` unchanged, inside and outside the span of the undone ones.
    LAMB's host-resident undo takes the saved trust ratios of the state."""
    from paper_2302_06173_b200 import LAMB
    lamb = kind == "lamb"
    kind = LAMB if lamb else kind
    h = OptimizerHyper(kind=LAMB, lr=1e-3, weight_decay=0.01) if lamb else HYP[kind]
    sizes = [1000, 77, 5000, 64, 3000, 12345]
    ref = DeviceState(sizes, dtype=dtype, kind=kind)
    seeded_fill_(ref.x, 1)
    seeded_fill_(ref.g, 2)
    seeded_fill_(ref.m, 3)
    if ref.v is not None:
        seeded_fill_(ref.v, 4)
        ref.v.abs_()
    ref.write_markers([(5, 0)] * len(sizes))
    ref.step(h)  # the pending update to undo (LAMB saves its trust ratios here)
    host = {k: getattr(ref, k).cpu().pin_memory() for k in ("x", "g", "m", "v") if getattr(ref, k) is not None}
    st = DeviceState(sizes, dtype=dtype, kind=kind, host_resident=True)
    assert st.x is None
    st.write_markers(ref.markers())
    if lamb:
        for i in range(len(sizes)):
            st.set_saved_scalars(i, ref.saved_scalars(i))
    out = {k: torch.zeros_like(v).pin_memory() for k, v in host.items() if k != "g"}
    st.undo_from_host(h, host, out, ids=ids, slice_elems=2000)
    torch.cuda.synchronize()
    ref.undo(h, ids)
    for k in out:  # undone groups bit-exact vs the device undo, the rest passed through
        assert torch.equal(out[k].cuda(), getattr(ref, k)), k
    assert st.markers() == ref.markers()
    with pytest.raises(RwError) as e:  # no device buffers: device-resident calls refuse
        st.undo(h, [2])
    assert e.value.name == "InvalidArgument"
    if lamb:
        assert [len(st.saved_scalars(i)) for i in ids] == [0] * len(ids)
    with pytest.raises(RwError) as e:  # guards before any copy
        st.undo_from_host(h, host, out, ids=[ids[-1]])
    assert e.value.name == "NothingToUndo"
    if not lamb:  # a device-resident state's own buffers are not the staging area
        dv = DeviceState(sizes, dtype=dtype, kind=kind)
        dv.write_markers([(6, 1)] * len(sizes))
        dv.undo_from_host(h, host, {k: torch.empty_like(v).pin_memory() for k, v in out.items()}, ids=ids,
                          slice_elems=2000)
        torch.cuda.synchronize()
        assert float(dv.x.abs().sum()) == 0.0


@pytest.mark.parametrize("cfg", ["adam340m", "adam1b"])
def test_full_size_configs_sampled_bitexact(restate, cfg):
    """The BASELINE sizes themselves (config 2 BERT-large 336M in 398 groups;
    the north-star 1B in 250 groups): step then undo in one launch each, every
    sampled element bit-identical to the fp32 restatement (elementwise ops, so
    sampling is exact), every marker as optimizer_step/undo leave it, and no
    non-finite value anywhere."""
    from paper_2302_06173_b200.workloads import CONFIGS
    sizes = CONFIGS[cfg]["sizes"]()
    st = DeviceState(sizes, kind=ADAM)
    seeded_fill_(st.x, 11)
    seeded_fill_(st.m, 12)
    st.m.mul_(0.01)
    seeded_fill_(st.v, 13)
    st.v.abs_().mul_(1e-4)
    seeded_fill_(st.g, 14)
    gen = torch.Generator(device="cuda").manual_seed(5)
    n = 1 << 20
    idx = torch.randint(0, st.total, (n,), device="cuda", generator=gen)
    x0, g0, m0, v0 = (getattr(st, k)[idx].cpu().numpy() for k in ("x", "g", "m", "v"))
    st.write_markers([(20, 0)] * len(sizes))
    h = HYP[ADAM]
    st.step(h)
    st.check_finite()
    assert st.markers() == [(21, 1)] * len(sizes)
    rx, rm, rv, _ = restate.step(ADAM, h, 20, x0, g0, m0, v0, dtype=np.float32)
    assert np.array_equal(_bits(st.x[idx].cpu().numpy()), _bits(rx))
    assert np.array_equal(_bits(st.m[idx].cpu().numpy()), _bits(rm))
    st.undo(h)
    st.check_finite()
    assert st.markers() == [(20, 0)] * len(sizes)
    ux, um, uv, _ = restate.undo(ADAM, h, 21, rx, g0, rm, rv, dtype=np.float32)
    assert np.array_equal(_bits(st.x[idx].cpu().numpy()), _bits(ux))
    assert np.array_equal(_bits(st.v[idx].cpu().numpy()), _bits(uv))


def test_group_beyond_2_pow_31_elements(restate):
    """Maximum-size edge case: one group of 2^31 + 4099 fp32 elements (x, g, m,
    v = 34 GB) plus a tiny trailing group — 64-bit offsets all the way through
    the work list, the TMA tiles and the marker; sampled elements bit-exact,
    both markers advanced."""
    n_big = (1 << 31) + 4099
    st = DeviceState([n_big, 33], kind=ADAM)
    for i, k in enumerate(("x", "g", "m", "v")):
        seeded_fill_(getattr(st, k), 60 + i)
    st.m.mul_(0.01)
    st.v.abs_().mul_(1e-4)
    st.write_markers([(3, 0), (3, 0)])
    gen = torch.Generator(device="cuda").manual_seed(1)
    idx = torch.cat([torch.randint(0, n_big, (1 << 18,), device="cuda", generator=gen),
                     torch.arange(n_big - 64, n_big, device="cuda"),          # the tail of the big group
                     torch.arange(st.offsets[1], st.offsets[1] + 33, device="cuda")])
    x0, g0, m0, v0 = (getattr(st, k)[idx].cpu().numpy() for k in ("x", "g", "m", "v"))
    h = HYP[ADAM]
    st.step(h)
    st.check_finite()
    assert st.markers() == [(4, 1), (4, 1)]
    rx, rm, rv, _ = restate.step(ADAM, h, 3, x0, g0, m0, v0, dtype=np.float32)
    assert np.array_equal(_bits(st.x[idx].cpu().numpy()), _bits(rx))
    assert np.array_equal(_bits(st.v[idx].cpu().numpy()), _bits(rv))
    st.undo(h)
    assert st.markers() == [(3, 0), (3, 0)]
    ux, um, uv, _ = restate.undo(ADAM, h, 4, rx, g0, rm, rv, dtype=np.float32)
    assert np.array_equal(_bits(st.x[idx].cpu().numpy()), _bits(ux))
    assert np.array_equal(_bits(st.m[idx].cpu().numpy()), _bits(um))


def test_empty_group_lists_are_noops():
    """step / undo / host-resident undo over no groups: OK, nothing changes
    (the batch extension of the one-block call; no launch, no marker write)."""
    sizes = [1000, 77, 5000]
    st = DeviceState(sizes, kind=ADAM)
    seeded_fill_(st.x, 1)
    seeded_fill_(st.g, 2)
    seeded_fill_(st.m, 3)
    seeded_fill_(st.v, 4)
    st.v.abs_()
    st.write_markers([(5, 0), (6, 1), (7, 0)])
    before = {k: getattr(st, k).clone() for k in ("x", "g", "m", "v")}
    mk = st.markers()
    h = HYP[ADAM]
    st.step(h, [])
    st.undo(h, [])
    host = {k: getattr(st, k).cpu().pin_memory() for k in ("x", "g", "m", "v")}
    out = {k: torch.empty_like(host[k]).pin_memory() for k in ("x", "m", "v")}
    st.undo_from_host(h, host, out, ids=[])
    torch.cuda.synchronize()
    assert st.markers() == mk
    for k, t in before.items():
        assert torch.equal(getattr(st, k), t), k

