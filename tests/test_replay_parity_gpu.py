"""Replay parity at the BASELINE config-4 depth with
DERIVED per-element tolerances, in two links:

(a) kernel == emulation.  Every GEMM of one stage 4096 -> 16384 -> 4096
    (make_stage, model.cpp:32-54) on a full config-4 micro-batch (R = 8 x 2048
    = 16384 rows: forward reduction depths K = 4096 / 16384, dgrad 16384 /
    4096, wgrad R = 16384) is compared with an fp64 evaluation of the SAME
    bf16 operands the kernel consumed (its own activations, dz and bf16 weight
    shadows) and the same epilogue.  Bound per element:
        |gpu - emu| <= ulp_bf16(out)                        (output rounding, x2 margin)
                     + L * 8 * sqrt(n) * 2^-24 * sum|terms|  (fp32 accumulation, probabilistic
                                                             bound, Higham & Mary, lambda = 8)
                     + 2^-10 * |y|                            (forward: tanh.approx.f32, 2^-11)
    L = Lipschitz constant of the epilogue (1 for tanh, |1 - y^2| for dtanh).
    A lost or duplicated K block moves an output by ~sqrt(64/n) of its size,
    i.e. many ulps: this is a tight check, not a 3e-2 * max bar.
    Sampled rows (forward, dgrad outputs) / sampled columns (wgrad, db).

(b) emulation == reference.  The reference library itself (oracle/_ref,
    fp64 triple loops, forward_stage / backward_stage, model.cpp:59-156) on
    three sampled rows of the same stage, against the GPU outputs, with a
    first-order statistical bound propagated from the bf16 roundings the B200
    path introduces (weights, y, dz, outputs: each a relative error uniform in
    [-2^-8, 2^-8], sigma = 2^-8/sqrt(3)); every element within 6 sigma and the
    RMS of err/sigma <= 1.5.

(c) one whole replayed iteration (2 stages, m = 4 micro-batches: forward,
    mse_loss, backward, accumulate_grads in ascending order, Adam step in
    reverse layer order; model.cpp:77-188) against the reference
    library running the same iteration, per block:
        ||g_gpu - g_ref|| <= 1e-2 ||g_ref||  for the accumulated gradients
        (each gradient element passes through <= 5 bf16 roundings of relative
        sigma 2^-8/sqrt(3): sqrt(5) * 2^-8/sqrt(3) = 5e-3, x2 margin), m and v
        within the same relative bound ((1-b1) g and (1-b2) g^2 are linear /
        quadratic in g), and the Adam update x_new - x_old within 3x it.
"""
import ctypes as C
import math

import numpy as np
import pytest
import torch

from oracle.oracle import _dptr
from paper_2302_06173_b200 import ADAM, OptimizerHyper
from paper_2302_06173_b200.replay import BoundaryLog, Stage, replay_group, synth_inputs

pytestmark = pytest.mark.gpu
U32 = 2.0 ** -24
LAM = 8.0
SIG = 2.0 ** -8 / math.sqrt(3.0)


def ulp_bf16(a: torch.Tensor) -> torch.Tensor:
    """Spacing of bf16 numbers at |a| (8-bit significand)."""
    a = a.abs().clamp_min(2.0 ** -126)
    return torch.exp2(torch.floor(torch.log2(a)) - 7)


def _assert_within(gpu: torch.Tensor, emu: torch.Tensor, bound: torch.Tensor, what: str):
    err = (gpu.double() - emu).abs()
    bad = err > bound
    ratio = (err / bound).max().item()
    assert not bad.any(), (f"{what}: {int(bad.sum())} of {bad.numel()} elements over the derived bound; "
                           f"max err/bound {ratio:.3g}, max err {err.max().item():.3g}")
    return ratio


def _dot_bound(n: int, mag: torch.Tensor, lip=1.0) -> torch.Tensor:
    return lip * LAM * math.sqrt(n) * U32 * mag


@pytest.fixture(scope="module")
def config4_stage():
    """One config-4 stage and a full micro-batch through forward + backward."""
    torch.manual_seed(0)
    R, dims, sid, seed = 16384, (4096, 16384, 4096), 1, 2302
    st = Stage(sid, dims[0], dims[1], dims[2], 2, seed, ADAM)
    x = synth_inputs(seed, 0, 0, R, dims[0])
    acts = st.new_acts(R, x)
    st.forward(acts)
    g = synth_inputs(seed, 1, 0, R, dims[2]).mul_(1e-3)  # a logged boundary gradient
    gout = torch.empty(R, dims[0], dtype=torch.bfloat16, device="cuda")
    st.backward(acts, g, gout, accumulate=False)
    torch.cuda.synchronize()
    s0, s1, _ = st._scr(R)  # after an L = 2 backward: s0 = dz of layer 1, s1 = dz of layer 0
    out = dict(R=R, dims=dims, sid=sid, seed=seed, st=st,
               x=acts[0].cpu(), y1=acts[1].cpu(), y2=acts[2].cpu(), g=g.cpu(), gout=gout.cpu(),
               dz2=s0[:R * dims[2]].view(R, dims[2]).cpu(), dz1=s1[:R * dims[1]].view(R, dims[1]).cpu(),
               W1=st.w16[0].view(dims[0], dims[1]).cpu(), W2=st.w16[1].view(dims[1], dims[2]).cpu(),
               b1=st.state.view("x", 1).cpu(), b2=st.state.view("x", 3).cpu(),
               dW1=st.grad_view(0).view(dims[0], dims[1]).cpu(), db1=st.grad_view(1).cpu(),
               dW2=st.grad_view(2).view(dims[1], dims[2]).cpu(), db2=st.grad_view(3).cpu())
    yield out
    del st
    torch.cuda.empty_cache()


ROWS = torch.tensor([0, 127, 128, 5000, 9999, 16383])   # tile edges and interior rows
COLS1 = torch.tensor([0, 1, 255, 256, 4095, 7777, 12000, 16383])
COLS2 = torch.tensor([0, 255, 256, 1023, 2048, 4095])


def test_forward_gemms_match_emulation_config4(config4_stage):
    c = config4_stage
    ratios = []
    for (xin, W, b, y, K, what) in ((c["x"], c["W1"], c["b1"], c["y1"], c["dims"][0], "forward layer 0 (K=4096)"),
                                    (c["y1"], c["W2"], c["b2"], c["y2"], c["dims"][1], "forward layer 1 (K=16384)")):
        X = xin[ROWS].double()
        Wd = W.double()
        s = X @ Wd + b.double()
        mag = X.abs() @ Wd.abs() + b.double().abs()
        ye = torch.tanh(s)
        bound = ulp_bf16(ye) + _dot_bound(K, mag) + 2.0 ** -10 * ye.abs() + 1e-30
        ratios.append(_assert_within(y[ROWS], ye, bound, what))
    assert max(ratios) > 0.0  # the comparison saw real data


def test_dtanh_first_bitexact(config4_stage):
    c = config4_stage
    g, y = c["g"].float(), c["y2"].float()
    dz = (g * (1.0 - y * y)).to(torch.bfloat16)  # fp32 ops in the kernel's order, then RNE to bf16
    assert torch.equal(dz.view(torch.int16), c["dz2"].view(torch.int16))


def test_dgrad_gemms_match_emulation_config4(config4_stage):
    c = config4_stage
    # layer 1 dgrad fused with layer 0's dtanh: dz1 = bf16(bf16(dz2 W2^T) * (1 - y1^2))
    dz2 = c["dz2"][ROWS].double()
    W2 = c["W2"].double()
    acc = dz2 @ W2.T
    mag = dz2.abs() @ W2.abs().T
    y1 = c["y1"][ROWS].double()
    lip = (1.0 - y1 * y1).abs()
    emu = acc * (1.0 - y1 * y1)
    bound = ulp_bf16(emu) + lip * (ulp_bf16(acc) + _dot_bound(c["dims"][2], mag)) + 4 * U32 * emu.abs() + 1e-30
    _assert_within(c["dz1"][ROWS], emu, bound, "dgrad layer 1 -> dz of layer 0 (K=4096)")
    # layer 0 dgrad = the stage's grad_out: bf16(dz1 W1^T), depth 16384
    dz1 = c["dz1"][ROWS].double()
    W1 = c["W1"].double()
    emu = dz1 @ W1.T
    mag = dz1.abs() @ W1.abs().T
    bound = ulp_bf16(emu) + _dot_bound(c["dims"][1], mag) + 1e-30
    _assert_within(c["gout"][ROWS], emu, bound, "dgrad layer 0 -> grad_out (K=16384)")


def test_wgrad_and_db_match_emulation_config4(config4_stage):
    c = config4_stage
    R = c["R"]
    for (xin, dz, dW, db, cols, what) in ((c["x"], c["dz1"], c["dW1"], c["db1"], COLS1, "layer 0"),
                                          (c["y1"], c["dz2"], c["dW2"], c["db2"], COLS2, "layer 1")):
        X = xin.double()
        D = dz[:, cols].double()
        emu = X.T @ D                       # dW[:, cols] = x^T dz over all R rows (model.cpp:121-131)
        mag = X.abs().T @ D.abs()
        _assert_within(dW[:, cols], emu, _dot_bound(R, mag) + 1e-30, f"wgrad {what} (depth R={R})")
        dbe = D.sum(0)                      # db = column sums of dz (model.cpp:132-137)
        _assert_within(db[cols], dbe, _dot_bound(R, D.abs().sum(0)) + 1e-30, f"db {what}")


def test_stage_vs_reference_library_config4_rows(ref, config4_stage):
    """Link (b): the reference's own forward_stage / backward_stage (fp64) on
    three rows of the config-4 stage, against the B200 outputs, within the
    propagated bf16 error model (6 sigma per element, RMS(err/sigma) <= 1.5)."""
    c = config4_stage
    rows = [0, 8191, 16383]
    din, dh, dout = c["dims"]
    rs = ref.L.ref_stage_make(c["sid"], din, dh, dout, 2, c["seed"])
    assert rs
    try:
        Wr = []
        for bi, n in enumerate((din * dh, dh, dh * dout, dout)):  # W0, b0, W1, b1 (fp64, as the reference holds them)
            w = np.empty(n)
            ref.L.ref_block_get(C.c_void_p(ref.L.ref_stage_block(rs, bi)), _dptr(w), None, None, None, None, None)
            Wr.append(torch.from_numpy(w))
        W1, b1 = Wr[0].view(din, dh), Wr[1]
        W2, b2 = Wr[2].view(dh, dout), Wr[3]
        x = c["x"][rows].double()
        yref = np.empty(len(rows) * dout)
        assert ref.L.ref_forward_stage(rs, _dptr(np.ascontiguousarray(x.numpy().ravel())), len(rows), din, 0,
                                       _dptr(yref)) == 0
        g = c["g"][rows].double()
        go_ref = np.empty(len(rows) * din)
        pg = [np.empty(n) for n in (din * dh, dh, dh * dout, dout)]
        parr = (C.POINTER(C.c_double) * 4)(*[_dptr(a) for a in pg])
        assert ref.L.ref_backward_stage(rs, _dptr(np.ascontiguousarray(g.numpy().ravel())), len(rows), dout, 0,
                                        _dptr(go_ref), parr) == 0
    finally:
        ref.L.ref_stage_free(rs)
    # reference intermediates (fp64) for the first-order propagation
    z1 = x @ W1 + b1
    y1 = torch.tanh(z1)
    z2 = y1 @ W2 + b2
    y2 = torch.tanh(z2)
    assert np.allclose(y2.numpy().ravel(), yref, rtol=0, atol=1e-12)  # fp64 restatement == _ref (sum order only)
    s2 = SIG * SIG
    v_z1 = s2 * ((x * x) @ (W1 * W1))                                 # W1 -> bf16
    v_y1 = (1 - y1 * y1) ** 2 * v_z1 + s2 * y1 * y1 + (2.0 ** -11) ** 2 / 3 * y1 * y1
    v_z2 = v_y1 @ (W2 * W2) + s2 * ((y1 * y1) @ (W2 * W2))           # y1 error, W2 -> bf16
    v_y2 = (1 - y2 * y2) ** 2 * v_z2 + s2 * y2 * y2 + (2.0 ** -11) ** 2 / 3 * y2 * y2
    sig_y2 = v_y2.sqrt()
    err = (c["y2"][rows].double() - torch.from_numpy(yref).view(len(rows), dout)).abs()
    assert (err <= 6 * sig_y2 + 1e-12).all(), f"forward vs _ref: max err/sigma {(err / sig_y2).max():.3g}"
    assert (err / sig_y2).pow(2).mean().sqrt() <= 1.5
    # backward: dz2 = g (1 - y2^2); dx1 = dz2 W2^T; dz1 = dx1 (1 - y1^2); grad_out = dz1 W1^T
    dz2 = g * (1 - y2 * y2)
    v_dz2 = (2 * g * y2) ** 2 * v_y2 + s2 * dz2 * dz2
    dx1 = dz2 @ W2.T
    v_dx1 = v_dz2 @ (W2 * W2).T + s2 * ((dz2 * dz2) @ (W2 * W2).T) + s2 * dx1 * dx1
    dz1 = dx1 * (1 - y1 * y1)
    v_dz1 = (1 - y1 * y1) ** 2 * v_dx1 + (2 * dx1 * y1) ** 2 * v_y1 + s2 * dz1 * dz1
    go = dz1 @ W1.T
    v_go = v_dz1 @ (W1 * W1).T + s2 * ((dz1 * dz1) @ (W1 * W1).T) + s2 * go * go
    assert np.allclose(go.numpy().ravel(), go_ref, rtol=1e-9, atol=1e-15)  # restatement == _ref
    sig = v_go.sqrt()
    err = (c["gout"][rows].double() - go).abs()
    assert (err <= 6 * sig + 1e-15).all(), f"grad_out vs _ref: max err/sigma {(err / sig).max():.3g}"
    assert (err / sig).pow(2).mean().sqrt() <= 1.5


def test_whole_replayed_iteration_vs_reference(ref):
    """Link (c): one whole iteration of a 2-stage group (both pipeline ends:
    synthetic inputs in, mse_loss out), m = 4, Adam from a warm state, through
    the B200 replay driver vs the reference library doing the same."""
    din, dh, dout, L, R, m, seed, it = 256, 1024, 256, 2, 512, 4, 77, 3
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    st = [Stage(s, din, dh, dout, L, seed, ADAM) for s in range(2)]
    rs = [ref.L.ref_stage_make(s, din, dh, dout, L, seed) for s in range(2)]
    rng = np.random.default_rng(5)
    hc = ref.hyper(dict(kind=ADAM, lr=1e-3, weight_decay=0.01, beta1=0.9, beta2=0.999, eps=1e-8))
    try:
        x_old = {}
        # warm optimizer state (fp32-representable, identical on both sides), t = 10
        for s in range(2):
            st[s].state.write_markers([(10, 0)] * (2 * L))
            for bi in range(2 * L):
                n = st[s].state.sizes[bi]
                mm = (rng.standard_normal(n) * 1e-3).astype(np.float32)
                vv = (np.abs(rng.standard_normal(n)) * 1e-6).astype(np.float32)
                st[s].state.view("m", bi).copy_(torch.from_numpy(mm))
                st[s].state.view("v", bi).copy_(torch.from_numpy(vv))
                blk = C.c_void_p(ref.L.ref_stage_block(rs[s], bi))
                ref.L.ref_block_set(blk, None, None, _dptr(mm.astype(np.float64)), _dptr(vv.astype(np.float64)), 10, 0)
                xr = np.empty(n)
                ref.L.ref_block_get(blk, _dptr(xr), None, None, None, None, None)
                x_old[(s, bi)] = xr
        # B200: one replayed iteration through the replay driver (first and last stage of the pipeline)
        replay_group(st, BoundaryLog(), it, it + 1, R, m, seed, h, first=True, last=True, dim=din)
        torch.cuda.synchronize()
        # reference: the same iteration, inputs = the bf16 values the B200 stage consumed
        per_mb = []
        for mb in range(m):
            x = synth_inputs(seed, it, mb, R, din).double().cpu().numpy().ravel()
            y0 = np.empty(R * dout)
            assert ref.L.ref_forward_stage(rs[0], _dptr(x), R, din, mb, _dptr(y0)) == 0
            y1 = np.empty(R * dout)
            assert ref.L.ref_forward_stage(rs[1], _dptr(y0), R, dout, mb, _dptr(y1)) == 0
            tgt = np.empty(R * dout)
            assert ref.L.ref_synth_targets(seed, it, mb, R, dout, _dptr(tgt)) == 0
            gl, loss = np.empty(R * dout), C.c_double()
            assert ref.L.ref_mse_loss(_dptr(y1), _dptr(tgt), R, dout, m, C.byref(loss), _dptr(gl)) == 0
            grads = {}
            go = np.empty(R * din)
            pg = [np.empty(n) for n in st[1].state.sizes]
            parr = (C.POINTER(C.c_double) * len(pg))(*[_dptr(a) for a in pg])
            assert ref.L.ref_backward_stage(rs[1], _dptr(gl), R, dout, mb, _dptr(go), parr) == 0
            grads[1] = pg
            go0 = np.empty(R * din)
            pg0 = [np.empty(n) for n in st[0].state.sizes]
            parr0 = (C.POINTER(C.c_double) * len(pg0))(*[_dptr(a) for a in pg0])
            assert ref.L.ref_backward_stage(rs[0], _dptr(go), R, dout, mb, _dptr(go0), parr0) == 0
            grads[0] = pg0
            per_mb.append(grads)
        for s in (1, 0):  # apply_layerwise_updates: stages and blocks in reverse layer order
            for bi in reversed(range(2 * L)):
                acc = ref.ordered_sum([per_mb[mb][s][bi] for mb in range(m)])  # accumulate_grads
                blk = C.c_void_p(ref.L.ref_stage_block(rs[s], bi))
                dims = st[s].dims
                shp = [dims[bi // 2], dims[bi // 2 + 1]] if bi % 2 == 0 else [dims[bi // 2 + 1]]  # W [in,out], b [out]
                shape = (C.c_size_t * len(shp))(*shp)
                assert ref.L.ref_optimizer_step(blk, _dptr(acc), shape, len(shp), C.byref(hc)) == 0
                n = acc.size
                xr, mr, vr = np.empty(n), np.empty(n), np.empty(n)
                ref.L.ref_block_get(blk, _dptr(xr), None, _dptr(mr), _dptr(vr), None, None)
                gg = st[s].grad_view(bi).cpu().double().numpy()
                xg = st[s].state.view("x", bi).cpu().double().numpy()
                mg = st[s].state.view("m", bi).cpu().double().numpy()
                vg = st[s].state.view("v", bi).cpu().double().numpy()
                rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)  # noqa: E731
                tag = f"stage {s} block {bi}"
                assert rel(gg, acc) <= 1e-2, (tag, "grad", rel(gg, acc))
                assert rel(mg, mr) <= 1e-2, (tag, "m", rel(mg, mr))
                assert rel(vg, vr) <= 1e-2, (tag, "v", rel(vg, vr))
                dx_ref = xr - x_old[(s, bi)]
                dx_gpu = xg - x_old[(s, bi)].astype(np.float32).astype(np.float64)
                assert rel(dx_gpu, dx_ref) <= 3e-2, (tag, "x update", rel(dx_gpu, dx_ref))
        for s in range(2):
            assert st[s].state.markers() == [(11, 0)] * (2 * L)
    finally:
        for r in rs:
            ref.L.ref_stage_free(r)
