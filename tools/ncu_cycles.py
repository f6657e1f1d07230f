"""Cycles per tcgen05.mma M128xN256xK16-equivalent from an ncu CSV of
tools/gemm_probe.cu (`--metrics sm__cycles_elapsed.max -k regex:umma_gemm --csv`)."""
import csv
import re
import statistics
import sys

SHAPES = {"<256, 0, 1, 1>": (16384, 16384, 4096), "<256, 0, 0, 2>": (16384, 4096, 16384),
          "<256, 1, 1, 4>": (4096, 16384, 16384), "<256, 0, 0, 0>": (16384, 16384, 4096)}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = {}
for r in rows[1:]:
    if not r[mi].startswith("sm__cycles_elapsed"):
        continue
    key = re.search(r"umma_gemm2?_kernel<[^>]*>", r[ki]).group(0)
    agg.setdefault(key, []).append(float(r[vi].replace(",", "")))
for key, v in agg.items():
    M, N, K = SHAPES[key[key.index("<"):]]
    print(f"{key:36s} {statistics.median(v) / (M * N * K / (128 * 256 * 16) / 148):7.1f} cycles/MMA  (n={len(v)})")
