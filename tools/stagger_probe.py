"""Does the relative placement of x, g, m, v change the 1B Adam undo rate?
Separate 4 GB allocations (4 GB apart: the streams the kernel reads side by
side are a power-of-two distance apart) vs one slab with a per-buffer
stagger.  usage: python tools/stagger_probe.py"""
import statistics
import sys
from pathlib import Path

sys.path.append(str(Path(__file__).resolve().parents[1]))  # a PYTHONPATH build variant wins
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2302_06173_b200 import ADAM, DeviceState, OptimizerHyper  # noqa: E402
from paper_2302_06173_b200.workloads import CONFIGS  # noqa: E402

h = OptimizerHyper(kind=ADAM, lr=1e-4, weight_decay=0.01)
for cfg in ("adam1b", "adam340m"):
    sizes = CONFIGS[cfg]["sizes"]()
    for rep in range(3):
        for stag in (None, 0, 4096, 65536 + 4096, (1 << 20) + 8192, 3 * (1 << 20) + 12288):
            st = DeviceState(sizes, kind=ADAM, stagger_bytes=stag)
            bench._fill_adam_state(st)
            st.write_markers([(10, 0)] * st.num_groups)
            nb = sum(sizes) * 28
            ts = []
            for i in range(8):
                st.step(h)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); st.undo(h); b.record()
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(a.elapsed_time(b))
            ptrs = [hex(t.data_ptr()) for t in (st.x, st.g, st.m, st.v)]
            print(cfg, rep, stag, round(nb / statistics.median(ts) / 1e6, 1), ptrs, flush=True)
            del st
            torch.cuda.empty_cache()
