"""Replay path on the GPU.

Bars:
  * forward_stage / backward_stage / mse_loss vs the fp64 reference library at
    desk shapes: |gpu - ref| <= 3e-2 * max|ref| per tensor, a smoke-level bar
    (the derived per-element bounds at config-4 depth live in
    tests/test_replay_parity_gpu.py);
  * logging replay == failure-free GPU ghost run, BIT FOR BIT (acceptance 4);
  * parallel recovery (mb mod d, ascending-mb merge) == sequential replay,
    BIT FOR BIT (acceptance 5), d = 2 emulated on one GPU;
  * MissingLogData when a needed record is absent.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle.oracle import _dptr
from paper_2302_06173_b200 import ADAM, SGDM, OptimizerHyper, RwError
from paper_2302_06173_b200.optim import ordered_sum
from paper_2302_06173_b200.replay import (BoundaryLog, Pipeline, Stage, helper_pass, mse_grad,
                                          parallel_assignment, replay_group, synth_inputs, synth_targets)

pytestmark = pytest.mark.gpu
TOL = 3e-2


def _close(gpu, ref, tol=TOL):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.max(np.abs(gpu - ref))
    scale = np.max(np.abs(ref))
    return err <= tol * scale + 1e-6, (err, scale)


@pytest.mark.parametrize("din,dh,dout,rows", [(64, 128, 64, 256),     # the desk shape
                                              (256, 1024, 256, 256),   # 4x expansion, K = 1024 accumulations
                                              (96, 200, 56, 100)])     # ragged: no dimension a tile multiple
def test_stage_forward_backward_vs_reference(ref, din, dh, dout, rows):
    torch.manual_seed(0)
    sid, L, seed = 1, 2, 2302
    st = Stage(sid, din, dh, dout, L, seed, ADAM)
    rs = ref.L.ref_stage_make(sid, din, dh, dout, L, seed)
    assert rs
    # identical initial parameters (fp32 master = single rounding of the reference's fp64)
    for bi in range(2 * L):
        blk = ref.L.ref_stage_block(rs, bi)
        n = st.state.sizes[bi]
        xr = np.empty(n)
        ref.L.ref_block_get(C.c_void_p(blk), _dptr(xr), None, None, None, None, None)
        assert np.array_equal(st.state.view("x", bi).cpu().numpy(), xr.astype(np.float32))
    x = synth_inputs(seed, 0, 0, rows, din)
    acts = st.new_acts(rows)
    acts[0].copy_(x)
    y = st.forward(acts)
    xin = x.float().cpu().numpy().astype(np.float64)
    yref = np.empty(rows * dout)
    assert ref.L.ref_forward_stage(rs, _dptr(np.ascontiguousarray(xin.ravel())), rows, din, 0, _dptr(yref)) == 0
    ok, info = _close(y.float().cpu().numpy().ravel(), yref)
    assert ok, info
    # backward: upstream gradient = mse grad against synthetic targets
    tgt = synth_targets(seed, 0, 0, rows, dout)
    g = mse_grad(y, tgt, 4)
    gref = np.empty(rows * dout)
    loss = C.c_double()
    assert ref.L.ref_mse_loss(_dptr(yref), _dptr(np.ascontiguousarray(tgt.cpu().numpy().astype(np.float64).ravel())),
                              rows, dout, 4, C.byref(loss), _dptr(gref)) == 0
    ok, info = _close(g.float().cpu().numpy().ravel(), gref)
    assert ok, info
    gin = np.ascontiguousarray(g.float().cpu().numpy().astype(np.float64).ravel())  # same upstream for both
    gout = torch.empty(rows, din, dtype=torch.bfloat16, device="cuda")
    st.backward(acts, g, gout, accumulate=False)
    gout_ref = np.empty(rows * din)
    pg = [np.empty(n) for n in st.state.sizes]
    parr = (C.POINTER(C.c_double) * len(pg))(*[_dptr(a) for a in pg])
    assert ref.L.ref_backward_stage(rs, _dptr(gin), rows, dout, 0, _dptr(gout_ref), parr) == 0
    ok, info = _close(gout.float().cpu().numpy().ravel(), gout_ref)
    assert ok, ("grad_out", info)
    for bi in range(2 * L):
        ok, info = _close(st.grad_view(bi).cpu().numpy(), pg[bi])
        assert ok, (bi, info)
    ref.L.ref_stage_free(rs)


def test_backward_is_deterministic():
    st = Stage(0, 64, 128, 64, 2, 7, ADAM)
    x = synth_inputs(7, 0, 0, 256, 64)
    acts = st.new_acts(256)
    acts[0].copy_(x)
    st.forward(acts)
    g = synth_inputs(7, 0, 1, 256, 64)
    outs = []
    for _ in range(3):
        gout = torch.empty(256, 64, dtype=torch.bfloat16, device="cuda")
        st.backward(acts, g, gout, accumulate=False)
        outs.append((gout.clone(), st.grad.clone()))
    for o in outs[1:]:
        assert torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1])


@pytest.mark.parametrize("rows,din,dh,dout", [(512, 256, 512, 256), (200, 96, 264, 56)])
def test_gemm_engines_agree_bitwise(rows, din, dh, dout):
    """The six GEMM engines (TMA-staged or register epilogue x single-CTA,
    CTA-pair or wide CTA-pair kernel) give the same bits for forward, backward
    with a fused stage boundary, and the accumulated fp32 weight gradients
    (second micro-batch: EPI_F32_ACC); the ragged shape exercises clipped TMA
    boxes (and, for the wide pair's 512-row tiles, whole out-of-range halves)."""
    from paper_2302_06173_b200.replay import LIB
    from paper_2302_06173_b200._lib import check
    results = []
    try:
        for epi, pair in ((1, 0), (0, 0), (1, 1), (0, 1), (1, 2), (0, 2)):
            check(LIB.rw_replay_set_gemm_engine(epi, pair))
            st = Stage(3, din, dh, dout, 2, 5, ADAM)
            prev = synth_inputs(5, 0, 9, rows, din)  # stands for the previous stage's output
            outs = []
            for mb in range(2):
                acts = st.new_acts(rows, synth_inputs(5, 0, mb, rows, din))
                st.forward(acts)
                g = synth_inputs(5, 1, mb, rows, dout)
                gout = torch.empty(rows, din, dtype=torch.bfloat16, device="cuda")
                # separate db pass on every engine (the register epilogue cannot fuse it)
                st.backward(acts, g, gout, accumulate=mb > 0, prev_y=prev, fuse_db=False)
                outs += [acts[1].clone(), acts[2].clone(), gout]
            torch.cuda.synchronize()
            results.append(outs + [st.grad.clone()])
    finally:
        check(LIB.rw_replay_set_gemm_engine(-1, -1))
    for other in results[1:]:
        for a, b in zip(results[0], other):
            assert torch.equal(a, b)


@pytest.mark.parametrize("pair", [0, 2])
def test_unaligned_outputs_take_the_register_epilogue(pair):
    """Output / y operands whose base is not 16-byte aligned cannot be TMA
    tensor-map operands: the GEMMs fall back to the register epilogue, whose
    vector accesses check the actual addresses.  The last layer's output, the
    stage-boundary gradient and the previous stage's y at a 2-byte offset give
    the same bits as aligned buffers."""
    from paper_2302_06173_b200.replay import LIB
    from paper_2302_06173_b200._lib import check
    rows, din, dh, dout = 200, 96, 264, 56
    check(LIB.rw_replay_set_gemm_engine(1, pair))
    try:
        def run(off):
            st = Stage(3, din, dh, dout, 2, 5, ADAM)
            prev_a = synth_inputs(5, 0, 9, rows, din)
            acts = st.new_acts(rows, synth_inputs(5, 0, 0, rows, din))
            last = torch.empty(rows * dout + 8, dtype=torch.bfloat16, device="cuda")[off:off + rows * dout]
            acts[-1] = last.view(rows, dout)
            st.forward(acts)
            gbuf = torch.empty(rows * din + 8, dtype=torch.bfloat16, device="cuda")[off:off + rows * din]
            pbuf = torch.empty(rows * din + 8, dtype=torch.bfloat16, device="cuda")[off:off + rows * din]
            pbuf.copy_(prev_a.reshape(-1))
            gout, prev = gbuf.view(rows, din), pbuf.view(rows, din)
            st.backward(acts, synth_inputs(5, 1, 0, rows, dout), gout, accumulate=False, prev_y=prev,
                        fuse_db=False)
            torch.cuda.synchronize()
            return [acts[1].clone(), acts[2].clone(), gout.clone(), st.grad.clone()]
        aligned, shifted = run(0), run(1)
        for a, b in zip(aligned, shifted):
            assert torch.equal(a, b)
    finally:
        check(LIB.rw_replay_set_gemm_engine(-1, -1))


@pytest.mark.parametrize("rows", [512, 4096, 200])
def test_fused_db_matches_separate_column_sums(rows):
    """db formed in the dgrad epilogue (per-32-row partials of the stored bf16
    dz, then the partial rows in order) vs the separate column-sum pass over
    dz: dW, grad_out and the last layer's db are the same bits; the fused
    layers' db agree to fp32 summation-order error."""
    st = Stage(2, 128, 512, 256, 3, 9, ADAM)
    prev = synth_inputs(9, 0, 7, rows, 128)
    res = []
    for fuse in (True, False):
        st.grad.zero_()
        outs = []
        for mb in range(2):
            acts = st.new_acts(rows, synth_inputs(9, 0, mb, rows, 128))
            st.forward(acts)
            gout = torch.empty(rows, 128, dtype=torch.bfloat16, device="cuda")
            st.backward(acts, synth_inputs(9, 1, mb, rows, 256), gout, accumulate=mb > 0, prev_y=prev,
                        fuse_db=fuse)
            outs.append(gout)
        torch.cuda.synchronize()
        res.append((outs, [st.grad_view(2 * l).clone() for l in range(3)],
                    [st.grad_view(2 * l + 1).clone() for l in range(3)]))
    (go_f, dw_f, db_f), (go_u, dw_u, db_u) = res
    for a, b in zip(go_f + dw_f, go_u + dw_u):
        assert torch.equal(a, b)
    assert torch.equal(db_f[2], db_u[2])  # the incoming dz: separate pass in both
    for l in (0, 1):
        scale = db_u[l].abs().max().item()
        assert (db_f[l] - db_u[l]).abs().max().item() <= 1e-5 * scale + 1e-7


@pytest.mark.parametrize("pair", [0, 1, 2])
def test_fused_db_partials_stay_inside_scratch(pair):
    """The per-32-row db partials are written for rows < M only: the tail
    boxes of a tile that hangs below the matrix (rows = 2100: the last 128-,
    256- or 512-row tile is mostly out of range) must not write past the
    ceil(rows / 32) partial rows the scratch holds."""
    from paper_2302_06173_b200.replay import LIB
    from paper_2302_06173_b200._lib import check
    rows = 2100
    check(LIB.rw_replay_set_gemm_engine(1, pair))
    try:
        st = Stage(2, 128, 512, 256, 3, 9, ADAM)
        mx = max(st.dims)
        need = (rows + 31) // 32 * mx
        big = torch.full((need + 64 * mx,), float("nan"), dtype=torch.float32, device="cuda")
        s0 = torch.empty(rows * mx, dtype=torch.bfloat16, device="cuda")
        s1 = torch.empty(rows * mx, dtype=torch.bfloat16, device="cuda")
        st._scratch[rows] = (s0, s1, big[:need])
        prev = synth_inputs(9, 0, 7, rows, 128)
        acts = st.new_acts(rows, synth_inputs(9, 0, 0, rows, 128))
        st.forward(acts)
        gout = torch.empty(rows, 128, dtype=torch.bfloat16, device="cuda")
        st.backward(acts, synth_inputs(9, 1, 0, rows, 256), gout, accumulate=False, prev_y=prev, fuse_db=True)
        torch.cuda.synchronize()
        assert torch.isnan(big[need:]).all(), "db partials written past the scratch"
        assert torch.isfinite(st.grad).all()
    finally:
        check(LIB.rw_replay_set_gemm_engine(-1, -1))


def _pipeline(kind=ADAM):
    h = OptimizerHyper(kind=kind, lr=1e-3 if kind == ADAM else 0.05, weight_decay=0.01)
    return Pipeline(p=3, dim=64, hidden=128, layers=2, rows=128, micro_batches=4, seed=11, kind=kind,
                    hyper=h), h


@pytest.mark.parametrize("kind", [ADAM, SGDM])
def test_logging_replay_equals_ghost_run_bitwise(kind):
    """§7 scenario at desk scale: checkpoint at it 2, failure at it 5, stage 1
    (a middle stage) replayed from logs -> bit-identical to the ghost run."""
    ghost, h = _pipeline(kind)
    log = BoundaryLog()
    snaps = {}
    for it in range(5):
        if it == 2:
            snaps = ghost.stages[1].snapshot()  # global checkpoint of the failed stage
        ghost.run_iteration(log_group=(1, 1), log=log)
    assert len(log.acts) == 5 * 4 and len(log.grads) == 5 * 4
    # replacement: fresh stage, load checkpoint, replay iterations 2..4
    rep = Stage(1, 64, 128, 64, 2, 11, kind)
    rep.restore(snaps)
    n = replay_group([rep], log, 2, 5, 128, 4, 11, h, first=False, last=False, dim=64)
    assert n == 3
    g = ghost.stages[1].state
    for name in ("x", "m", "v"):
        a, b = getattr(rep.state, name), getattr(g, name)
        if a is None:
            continue
        assert torch.equal(a.view(torch.int32), b.view(torch.int32)), name
    assert rep.state.markers() == g.markers()


def test_logging_replay_equals_ghost_run_config4_shapes():
    """The same acceptance property at config-4 sizes (stages
    4096 -> 16384 -> 4096, micro-batch 8 x 2048 = 16384 rows), on a 3-stage
    pipeline with 2 micro-batches: the middle stage replayed from its logs
    over 2 iterations equals the ghost run bit for bit (x, m, v, markers)."""
    h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
    rows, m = 16384, 2
    ghost = Pipeline(p=3, dim=4096, hidden=16384, layers=2, rows=rows, micro_batches=m, seed=23, kind=ADAM,
                     hyper=h)
    log = BoundaryLog()
    snap = ghost.stages[1].snapshot()
    for it in range(2):
        ghost.run_iteration(log_group=(1, 1), log=log)
    rep = Stage(1, 4096, 16384, 4096, 2, 23, ADAM)
    rep.restore(snap)
    assert replay_group([rep], log, 0, 2, rows, m, 23, h, first=False, last=False, dim=4096) == 2
    g = ghost.stages[1].state
    for name in ("x", "m", "v"):
        assert torch.equal(getattr(rep.state, name).view(torch.int32), getattr(g, name).view(torch.int32)), name
    assert rep.state.markers() == g.markers()
    del ghost, rep, log
    torch.cuda.empty_cache()


def test_group_replay_last_stages_bitwise():
    ghost, h = _pipeline()
    log = BoundaryLog(pinned=True)  # logs in pinned host memory
    for it in range(3):
        if it == 1:
            s1, s2 = ghost.stages[1].snapshot(), ghost.stages[2].snapshot()
        ghost.run_iteration(log_group=(1, 2), log=log)
    assert len(log.grads) == 0  # the last stage's gradient comes from the loss, never logged
    a, b = Stage(1, 64, 128, 64, 2, 11, ADAM), Stage(2, 64, 128, 64, 2, 11, ADAM)
    a.restore(s1)
    b.restore(s2)
    replay_group([a, b], log, 1, 3, 128, 4, 11, h, first=False, last=True, dim=64)
    assert torch.equal(a.state.x, ghost.stages[1].state.x)
    assert torch.equal(b.state.x, ghost.stages[2].state.x)
    assert torch.equal(b.state.v, ghost.stages[2].state.v)


def test_parallel_recovery_equals_sequential_bitwise():
    ghost, h = _pipeline()
    log = BoundaryLog()
    for it in range(3):
        if it == 1:
            snap = ghost.stages[1].snapshot()
        ghost.run_iteration(log_group=(1, 1), log=log)
    seq = Stage(1, 64, 128, 64, 2, 11, ADAM)
    seq.restore(snap)
    replay_group([seq], log, 1, 3, 128, 4, 11, h, first=False, last=False, dim=64)
    # d = 2 helpers (emulated in-process): Fig 6 assignment {0,2} / {1,3}
    assert parallel_assignment(4, 2) == [[0, 2], [1, 3]]
    helpers = [Stage(1, 64, 128, 64, 2, 11, ADAM) for _ in range(2)]
    for hs in helpers:
        hs.restore(snap)
    for it in range(1, 3):
        per_mb = {}
        for r, hs in enumerate(helpers):
            per_mb.update(helper_pass([hs], log, it, parallel_assignment(4, 2)[r], 128, 4, 11, False, False, 64))
        merged = ordered_sum([per_mb[mb][0] for mb in range(4)])
        for hs in helpers:
            hs.step(h, grad=merged)
    for hs in helpers:
        assert torch.equal(hs.state.x, seq.state.x)
        assert torch.equal(hs.state.m, seq.state.m)
        assert torch.equal(hs.state.v, seq.state.v)
    assert torch.equal(seq.state.x, ghost.stages[1].state.x)


def test_missing_log_raises():
    ghost, h = _pipeline()
    log = BoundaryLog()
    snap = ghost.stages[1].snapshot()
    ghost.run_iteration(log_group=(1, 1), log=log)
    del log.grads[(0, 2)]
    rep = Stage(1, 64, 128, 64, 2, 11, ADAM)
    rep.restore(snap)
    with pytest.raises(RwError) as e:
        replay_group([rep], log, 0, 1, 128, 4, 11, h, first=False, last=False, dim=64)
    assert e.value.name == "MissingLogData"


def test_training_loss_decreases():
    ghost, h = _pipeline()
    losses = [ghost.run_iteration() for _ in range(8)]
    assert all(np.isfinite(losses)) and losses[-1] < losses[0]


def test_middle_group_fused_boundaries_bitwise():
    """A 3-stage middle group (stages 1..3 of 5) replayed on one GPU: the two
    group-internal boundaries use the fused dgrad -> previous-stage dz epilogue
    (rw_stage_backward_ex); sequential replay and two parallel helpers must
    both equal the ghost run (which exchanges bf16 gradients between stages)
    bit for bit."""
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    ghost = Pipeline(p=5, dim=64, hidden=96, layers=2, rows=160, micro_batches=4, seed=3, kind=ADAM, hyper=h)
    log = BoundaryLog()
    for it in range(3):
        if it == 1:
            snaps = [ghost.stages[s].snapshot() for s in (1, 2, 3)]
        ghost.run_iteration(log_group=(1, 3), log=log)
    mk = lambda: [Stage(s, 64, 96, 64, 2, 3, ADAM) for s in (1, 2, 3)]  # noqa: E731
    seq = mk()
    for st, sn in zip(seq, snaps):
        st.restore(sn)
    replay_group(seq, log, 1, 3, 160, 4, 3, h, first=False, last=False, dim=64)
    helpers = [mk(), mk()]
    for grp in helpers:
        for st, sn in zip(grp, snaps):
            st.restore(sn)
    for it in range(1, 3):
        per_mb = {}
        for r, grp in enumerate(helpers):
            per_mb.update(helper_pass(grp, log, it, parallel_assignment(4, 2)[r], 160, 4, 3, False, False, 64))
        for k in range(3):
            merged = ordered_sum([per_mb[mb][k] for mb in range(4)])
            for grp in helpers:
                grp[k].step(h, grad=merged)
    for k, s in enumerate((1, 2, 3)):
        g = ghost.stages[s].state
        for name in ("x", "m", "v"):
            assert torch.equal(getattr(seq[k].state, name), getattr(g, name)), (s, name)
            for grp in helpers:
                assert torch.equal(getattr(grp[k].state, name), getattr(g, name)), (s, name)
