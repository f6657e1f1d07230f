"""The resolver's decisions executed on the device (recovery.apply_resolution),
single survivor: a torn update (MidUpdate(k)) is resolved by
  * undo  -> every group back at t, bit-identical to the state before the step
             re-stepped (the undo of each group is exact w.r.t. optimizer_undo);
  * redo  -> the lagging groups stepped with the cached gradient: bit-identical
             to an uninterrupted step of all groups;
and AMSGrad (not invertible) is forced onto redo."""
import pytest
import torch

from paper_2302_06173_b200 import ADAM, AMSGRAD, DeviceState, OptimizerHyper, seeded_fill_
from paper_2302_06173_b200.recovery import apply_resolution, resolve

pytestmark = pytest.mark.gpu
SIZES = [3000, 5000, 700, 12000]


def _state(kind):
    st = DeviceState(SIZES, kind=kind)
    for i, n in enumerate(("x", "g", "m", "v")):
        seeded_fill_(getattr(st, n), 70 + i)
    st.v.abs_()
    st.write_markers([(7, 0)] * len(SIZES))
    return st


@pytest.mark.parametrize("kind", [ADAM, AMSGRAD])
def test_redo_equals_uninterrupted_step(kind):
    h = OptimizerHyper(kind=kind, lr=1e-3, weight_decay=0.01)
    grad = torch.empty_like(_state(kind).x)
    seeded_fill_(grad, 99)
    full = _state(kind)
    full.step(h, grad=grad)
    torn = _state(kind)
    torn.step(h, grad=grad, stop_after=3)          # groups 3, 2, 1 updated; group 0 lagging
    mk = torn.markers()
    assert mk == [(7, 0), (8, 1), (8, 1), (8, 1)]
    plan = resolve(mk, h, lens=SIZES, grad_ready=[True] * 4, policy="min_cost" if kind == ADAM else "undo")
    assert plan.strategy == "Redo" and plan.redo_ids == [0] and plan.target == 8
    apply_resolution(torn, h, plan, grad=grad)
    assert torn.markers() == full.markers()
    for n in ("x", "m", "v"):
        assert torch.equal(getattr(torn, n), getattr(full, n)), n


def test_undo_returns_every_group_to_t():
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    torn = _state(ADAM)
    torn.step(h, stop_after=2)                      # groups 3, 2 updated
    plan = resolve(torn.markers(), h, lens=SIZES)
    assert plan.strategy == "Undo" and sorted(plan.undo_ids) == [2, 3]
    apply_resolution(torn, h, plan)
    assert torn.markers() == [(7, 0)] * 4
    # stepping everything again from the resolved state == stepping the original state
    again = _state(ADAM)
    torn.step(h)
    again.step(h)
    for n in ("x", "m", "v"):
        a, b = getattr(torn, n), getattr(again, n)
        assert torch.allclose(a, b, rtol=1e-6, atol=1e-7), n
