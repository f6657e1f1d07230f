"""Generate tests/golden/*.json from the REFERENCE library itself
(oracle/_ref/librewind_ref.so, built from /root/reference by oracle/Makefile).

Run here (the reference is not on the GPU box):  python tests/golden/make_golden.py
Floats are stored as hex strings (float.hex) so the fixtures are bit-exact.

Contents
  spec:   the SPEC known-answer vectors listed in SURVEY.md §4
  blocks: per optimizer kind, a seeded 67-element fp64 block (ragged: not a
          multiple of the vector width) with its state after step and after
          undo, produced by rewind::optimizer_step / optimizer_undo.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import ADAM, ADAMW, AMSGRAD, SGD, SGDM, Ref, RefError  # noqa: E402

H = lambda a: [float(v).hex() for v in np.asarray(a, np.float64).ravel()]  # noqa: E731


def main():
    ref = Ref()
    spec = {}
    # SPEC:109  SGD x=[2], g=[1], eta=0.1, wd=0.01
    b = ref.block(1)
    b.set(x=[2.0], g=[0.0], m=[0.0], v=[0.0])
    hs = dict(kind=SGD, lr=0.1, weight_decay=0.01)
    b.step(np.array([1.0]), hs)
    spec["sgd_step"] = H(b.get()["x"])
    b.undo(hs)
    spec["sgd_undo"] = H(b.get()["x"])
    try:  # SPEC:133 undo after undo
        b.undo(hs)
        spec["double_undo"] = "OK"
    except RefError as e:
        spec["double_undo"] = e.name
    # SPEC:110 SGDM
    b = ref.block(1)
    b.set(x=[1.0], g=[0.0], m=[0.0], v=[0.0])
    hm = dict(kind=SGDM, lr=0.1, momentum=0.9, dampening=0.0)
    b.step(np.array([1.0]), hm)
    st = b.get()
    spec["sgdm_step_m"], spec["sgdm_step_x"] = H(st["m"]), H(st["x"])
    # SPEC:116 SGDM mu=0 undo -> NonInvertibleHyper
    b = ref.block(1)
    b.set(x=[1.0], g=[0.0], m=[0.0], v=[0.0])
    h0 = dict(kind=SGDM, lr=0.1, momentum=0.0)
    b.step(np.array([1.0]), h0)
    try:
        b.undo(h0)
        spec["sgdm_mu0_undo"] = "OK"
    except RefError as e:
        spec["sgdm_mu0_undo"] = e.name
    # SPEC:116/128 AMSGrad
    b = ref.block(1)
    try:
        b.step(np.array([1.0]), dict(kind=AMSGRAD, require_invertible=True))
        spec["amsgrad_require_invertible"] = "OK"
    except RefError as e:
        spec["amsgrad_require_invertible"] = e.name
    b.step(np.array([1.0]), dict(kind=AMSGRAD))
    try:
        b.undo(dict(kind=AMSGRAD))
        spec["amsgrad_undo"] = "OK"
    except RefError as e:
        spec["amsgrad_undo"] = e.name
    spec["l2_norm_3_4"] = float(ref.l2_norm([3.0, 4.0])).hex()
    spec["bubble_4_4"] = list(ref.bubble_ratio(4, 4))
    spec["bubble_8_4"] = list(ref.bubble_ratio(8, 4))
    spec["grid_4_4"] = ref.schedule_grid(4, 4)
    spec["seeded_fill_2x2_7"] = H(ref.seeded_fill(4, 7))
    spec["crc32_123456789"] = ref.crc32(b"123456789")
    spec["derive_seed_2302_0_1"] = str(ref.derive_seed(2302, [0, 1]))

    blocks = {}
    hypers = {
        "sgd": dict(kind=SGD, lr=0.05, weight_decay=0.01),
        "sgdm": dict(kind=SGDM, lr=0.1, momentum=0.9, dampening=0.1, weight_decay=1e-4),
        "adam": dict(kind=ADAM, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01),
        "adamw": dict(kind=ADAMW, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01),
    }
    n = 67
    for ki, (name, h) in enumerate(hypers.items()):
        b = ref.block(n, seed=1000 + ki)
        x0 = b.get()["x"]
        g0 = ref.seeded_fill(n, 2000 + ki)
        m0 = ref.seeded_fill(n, 3000 + ki) * 0.5
        v0 = np.abs(ref.seeded_fill(n, 4000 + ki)) * 0.01
        t0 = 3
        b.set(x=x0, g=np.zeros(n), m=m0, v=v0, t=t0, updated=False)
        b.step(g0, h)
        s1 = b.get()
        b.undo(h)
        s2 = b.get()
        blocks[name] = dict(hyper=h, t0=t0, x0=H(x0), g=H(g0), m0=H(m0), v0=H(v0),
                            step=dict(x=H(s1["x"]), m=H(s1["m"]), v=H(s1["v"]), t=s1["t"]),
                            undo=dict(x=H(s2["x"]), m=H(s2["m"]), v=H(s2["v"]), t=s2["t"]))
    out = ROOT / "tests" / "golden" / "spec_vectors.json"
    out.write_text(json.dumps(dict(spec=spec, blocks=blocks), indent=1))
    print("wrote", out)


if __name__ == "__main__":
    main()
