"""Profiling driver: Adam step+undo over the config-2 (BERT-large) fp32 state,
through the C ABI.  optim_kernel launches alternate step, undo, step, undo...
so `ncu -k regex:optim_kernel -s 3 -c 1` captures an undo launch."""
import sys
from pathlib import Path

sys.path.append(str(Path(__file__).resolve().parents[1]))  # a PYTHONPATH build variant wins

import torch  # noqa: E402

from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper, seeded_fill_  # noqa: E402
from paper_2302_06173_b200.workloads import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "adam340m"
dtype = torch.float64 if (len(sys.argv) > 2 and sys.argv[2] == "f64") else torch.float32
sizes = CONFIGS[cfg]["sizes"]()
st = DeviceState(sizes, dtype=dtype, kind=ADAM)
for i, t in enumerate((st.x, st.g, st.m, st.v)):
    seeded_fill_(t, 10 + i)
st.m.mul_(0.01)
st.v.abs_().mul_(1e-4)
h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
st.write_markers([(10, 0)] * len(sizes))
for _ in range(3):
    st.step(h)
    st.undo(h)
torch.cuda.synchronize()
st.check_finite()
print("prof_undo done", cfg, dtype)
