"""How much of the 1B Adam undo's throughput is lost to the board's power cap
in a back-to-back step/undo loop?  Times each undo after an idle gap of g ms
(the GPU rests, as it does during failure detection before a real recovery's
single undo) with nvidia-smi power/clock sampling.
usage: python tools/undo_gap_probe.py"""
import statistics
import sys
import time
from pathlib import Path

sys.path.append(str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper  # noqa: E402
from paper_2302_06173_b200.workloads import CONFIGS  # noqa: E402
import bench  # noqa: E402

h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
sizes = CONFIGS["adam1b"]["sizes"]()
st = DeviceState(sizes, kind=ADAM)
bench._fill_adam_state(st)
st.write_markers([(10, 0)] * st.num_groups)
nb = sum(sizes) * 28
for _ in range(3):
    st.step(h)
    st.undo(h)
torch.cuda.synchronize()
for gap_ms in (0, 2, 10, 50, 200, 0):
    ts = []
    with bench.ClockSampler(0) as clk:
        for i in range(10):
            st.step(h)
            torch.cuda.synchronize()
            if gap_ms:
                time.sleep(gap_ms / 1e3)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            st.undo(h)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
    m = statistics.median(ts)
    print(f"gap {gap_ms:4d} ms: undo {m:.4f} ms = {nb / m / 1e6:.1f} GB/s  min {min(ts):.4f}  clocks {clk.summary()}",
          flush=True)
