"""Sustained (power-capped) bf16 GEMM throughput: this repo's tcgen05 GEMM
(through rw_stage_forward: 4096 -> 16384 -> 4096, bias + tanh fused, 16384
rows) against cuBLAS (torch.matmul, same two products, no epilogue), each
run back to back for ~`secs` seconds with nvidia-smi clocks / power sampled.
Set RW_GEMM_PAIR=1 for the CTA-pair kernel.

    python tools/sustained_gemm.py [secs]
"""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.append(str(Path(__file__).resolve().parents[1]))  # a PYTHONPATH build variant wins

import torch  # noqa: E402

from paper_2302_06173_b200 import ADAM  # noqa: E402  (before bench, which puts the repo first on sys.path)
from paper_2302_06173_b200.replay import Stage, synth_inputs  # noqa: E402
from bench import ClockSampler  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
R, D, H = 16384, 4096, 16384
flop = 2 * (2.0 * R * D * H)
st = Stage(0, D, H, D, 2, 2302, ADAM)
x = synth_inputs(5, 0, 0, R, D)
acts = st.new_acts(R, x)
w1 = torch.randn(D, H, device="cuda", dtype=torch.bfloat16)
w2 = torch.randn(H, D, device="cuda", dtype=torch.bfloat16)
h = torch.empty(R, H, device="cuda", dtype=torch.bfloat16)
y = torch.empty(R, D, device="cuda", dtype=torch.bfloat16)


def ours():
    st.forward(acts)


def cublas():
    torch.matmul(x, w1, out=h)
    torch.matmul(h, w2, out=y)


out = {}
for name, fn in (("ours", ours), ("cublas", cublas), ("ours_again", ours)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    # calibrate the count for ~secs seconds
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    n = max(10, int(secs / ((time.perf_counter() - t0) / 10)))
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    pw = []
    for ln in clk.lines:
        p = [q.strip() for q in ln.split(",")]
        try:
            pw.append(float(p[3]))
        except (IndexError, ValueError):
            pass
    out[name] = dict(ms_per_pass=round(ms, 3), tflops=round(flop / (ms * 1e-3) / 1e12, 1), passes=n,
                     clocks=clk.summary(), power_w_median=statistics.median(pw) if pw else None)
print(json.dumps(out, indent=1))
