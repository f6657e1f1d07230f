"""Real crash -> detect -> repair -> recover on 2 B200s (tools/real_failure.py):
the survivor aborts its NCCL communicator, a replacement process joins the
next generation on the freed GPU and receives the resolved state bit for bit
(device CRC32 of x, m, v + markers)."""
import os
import subprocess
import sys
import json
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_real_crash_recovery_two_gpus():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "real_failure.py"), "small"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=dict(os.environ))
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and line, r.stderr[-2000:]
    out = json.loads(line[-1])
    assert out["crashed_rank_exit"] == 1 and out["replacement_rank"] == 1
    assert out["strategy"] == "Undo" and out["undo_groups"] == 12
    assert out["identical"], out
