"""Kernel times of the GPU CRC32 (rw_crc32_device) on a 134 MB record."""
import ctypes as C
import sys
from pathlib import Path

sys.path.append(str(Path(__file__).resolve().parents[1]))  # a PYTHONPATH build variant wins
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2302_06173_b200._lib import LIB, check  # noqa: E402

x = torch.randint(0, 255, (134217728,), dtype=torch.uint8, device="cuda")
out = torch.zeros(1, dtype=torch.int32, device="cuda")
sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    check(LIB.rw_crc32_device(C.c_void_p(x.data_ptr()), x.numel(), C.c_void_p(out.data_ptr()), sh))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        check(LIB.rw_crc32_device(C.c_void_p(x.data_ptr()), x.numel(), C.c_void_p(out.data_ptr()), sh))
    torch.cuda.synchronize()
for e in prof.events():
    if e.device_type.name == "CUDA":
        print(f"{e.name[:60]:60s} {(e.time_range.end - e.time_range.start):9.1f} us")

# event-timed windows of 10 calls (as bench.logging_bench) and host time per call
import time  # noqa: E402
for w in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(10):
        check(LIB.rw_crc32_device(C.c_void_p(x.data_ptr()), x.numel(), C.c_void_p(out.data_ptr()), sh))
    e1.record()
    th = (time.perf_counter() - t0) / 10 * 1e3
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"window {w}: {ms:.3f} ms per call on the GPU timeline = {x.numel() / ms / 1e6:.0f} GB/s, host {th:.3f} ms per call")
