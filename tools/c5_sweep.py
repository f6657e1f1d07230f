"""Config 5: selective-logging sweep (bench.config5_sweep) on its own.
usage: python tools/c5_sweep.py [m] [out.json]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/c5_sweep.json"
res = bench.config5_sweep(m)
Path(out).parent.mkdir(exist_ok=True)
Path(out).write_text(json.dumps(res, indent=1))
print(json.dumps(res["sweep"], indent=1))
