"""SPEC acceptance 4, 6 and 7: logging-based recovery at
desk scale, through the product path (tcgen05 replay GEMMs, the native
upstream-backup Logger writing SWFT chunk files, the native checkpoint store
and log GC).

Setup (the SPEC section 7 scenario): an 8-stage pipeline folded onto 4
simulated machines of 2 stages each (cuts at stages 2, 4, 6).  Every message
that crosses a machine boundary is logged by its SENDER machine (upstream
backup), each machine with its own Logger into one shared log
directory; the global checkpoint is one worker per machine, committed by a
single manifest.

* Acceptance 4: ckpt@100, kill@150.  The failed machine's replacement loads
  the checkpoint, replays from the logs, and must equal the failure-free
  ghost run bit for bit at iteration 150 (x, m, v, markers); exactly 50
  iterations are replayed; the survivors' parameters are untouched.
* Acceptance 6: 50 randomized single-machine failure points with checkpoints
  every 6 iterations, small chunks (5 records) and GC after every checkpoint:
  the committed + flushed logs always hold every inbound message the replay
  needs (zero MissingLogData), and every replay equals the ghost bit for bit.
* Acceptance 7: after the GC at checkpoint c no live chunk has max iteration
  < c, and the live log payload never exceeds T x the per-iteration boundary
  bytes (T = checkpoint interval).
"""
import glob
import os
import random

import pytest
import torch

from paper_2302_06173_b200 import ADAM, OptimizerHyper
from paper_2302_06173_b200 import logstore
from paper_2302_06173_b200.checkpoint import commit_checkpoint, gc_logs, latest_checkpoint, load_checkpoint, \
    write_checkpoint
from paper_2302_06173_b200.replay import Pipeline, Stage, replay_group

pytestmark = pytest.mark.gpu

P, MACHINES = 8, 4
PER = P // MACHINES
CUTS = [PER * k for k in range(1, MACHINES)]
DIM, HID, LAYERS, ROWS, MB, SEED = 64, 128, 2, 128, 4, 11
H = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)


def _stages_of(machine):
    return list(range(machine * PER, (machine + 1) * PER))


def _checkpoint(ghost, ckpt_dir, it):
    for k in range(MACHINES):
        write_checkpoint([ghost.stages[s].state for s in _stages_of(k)], ckpt_dir, it, worker=k, commit=False)
    commit_checkpoint(ckpt_dir, it, MACHINES)


def _recover(failed, ckpt_dir, log_dir, fail_it):
    """recover_replay of one failed machine: fresh stages, the
    latest committed checkpoint, the inbound logs from the survivors' files."""
    stages = [Stage(s, DIM, HID, DIM, LAYERS, SEED + 99, ADAM) for s in _stages_of(failed)]  # other init
    c, _ = load_checkpoint([st.state for st in stages], ckpt_dir, iteration=latest_checkpoint(ckpt_dir),
                           worker=failed)
    for st in stages:
        st.refresh_shadows()
    first, last = _stages_of(failed)[0], _stages_of(failed)[-1]
    logs = logstore.load_log_dir(log_dir, receivers={first, last}, min_iteration=c)
    n = replay_group(stages, logs, c, fail_it, ROWS, MB, SEED, H, first=failed == 0,
                     last=failed == MACHINES - 1, dim=DIM)
    return stages, c, n


def _equal_to_ghost(stages, ghost, failed):
    for st, s in zip(stages, _stages_of(failed)):
        g = ghost.stages[s].state
        for name in ("x", "m", "v"):
            if not torch.equal(getattr(st.state, name), getattr(g, name)):
                return False
        if st.state.markers() != g.markers():
            return False
    return True


def _digest(ghost, machines):
    return {s: [getattr(ghost.stages[s].state, n).clone() for n in ("x", "m", "v")]
            for k in machines for s in _stages_of(k)}


@pytest.mark.parametrize("failed", [1, 3])
def test_acceptance4_ckpt100_kill150(tmp_path, failed):
    log_dir, ckpt_dir = str(tmp_path / "logs"), str(tmp_path / "ck")
    ghost = Pipeline(p=P, dim=DIM, hidden=HID, layers=LAYERS, rows=ROWS, micro_batches=MB, seed=SEED, kind=ADAM,
                     hyper=H)
    loggers = {k: logstore.Logger(log_dir, machine=k, chunk_records=64, pinned_bytes=8 << 20)
               for k in range(MACHINES)}
    for it in range(150):
        if it == 100:
            for lg in loggers.values():
                lg.flush()
            _checkpoint(ghost, ckpt_dir, 100)
            gc_logs(log_dir, ckpt_dir, 100)
        ghost.run_iteration(cuts=CUTS, senders=loggers)
    # kill@150: the failed machine's state is gone; its neighbours flush what they sent it
    for k, lg in loggers.items():
        if k != failed:
            lg.flush()
    survivors = [k for k in range(MACHINES) if k != failed]
    before = _digest(ghost, survivors)
    stages, c, n = _recover(failed, ckpt_dir, log_dir, 150)
    assert (c, n) == (100, 50)  # exactly 50 iterations replayed
    assert _equal_to_ghost(stages, ghost, failed)
    after = _digest(ghost, survivors)  # survivors untouched by the recovery
    assert all(torch.equal(a, b) for s in before for a, b in zip(before[s], after[s]))
    for lg in loggers.values():
        lg.close()


def _live_chunks(log_dir):
    out = []
    for path in sorted(glob.glob(os.path.join(log_dir, "m*.swft"))):
        its = [int(r.iteration) for r, _ in logstore.read_chunk(path)]
        out.append((path, max(its), sum(1 for _ in its)))
    return out


def test_acceptance6_and_7_random_failures_chunking_gc(tmp_path):
    log_dir, ckpt_dir = str(tmp_path / "logs"), str(tmp_path / "ck")
    T, ITERS, POINTS = 6, 36, 50
    rng = random.Random(2302)
    # failure points: (iteration, machine), sorted; a point at f is checked
    # right after iteration f-1 completes (survivors at iteration f)
    points = sorted((rng.randint(1, ITERS), rng.randrange(MACHINES)) for _ in range(POINTS))
    ghost = Pipeline(p=P, dim=DIM, hidden=HID, layers=LAYERS, rows=ROWS, micro_batches=MB, seed=SEED, kind=ADAM,
                     hyper=H)
    loggers = {k: logstore.Logger(log_dir, machine=k, chunk_records=5, pinned_bytes=8 << 20)
               for k in range(MACHINES)}
    rec_bytes = ROWS * DIM * 2  # one bf16 boundary tensor
    per_iter = len(CUTS) * 2 * MB * rec_bytes  # act + grad across each cut, per micro-batch
    missing = replays = 0
    pi = 0
    for it in range(ITERS + 1):
        while pi < len(points) and points[pi][0] == it:
            failed = points[pi][1]
            for k, lg in loggers.items():
                if k != failed:
                    lg.flush()  # the survivors' committed + flushed logs
            try:
                stages, c, n = _recover(failed, ckpt_dir, log_dir, it)
            except Exception as e:  # noqa: BLE001
                if "MissingLogData" in str(e):
                    missing += 1
                    pi += 1
                    continue
                raise
            assert n == it - c and 0 <= n <= T
            assert _equal_to_ghost(stages, ghost, failed), (it, failed)
            replays += 1
            pi += 1
        if it == ITERS:
            break
        if it % T == 0:
            for lg in loggers.values():
                lg.flush()
            # acceptance 7: just before the checkpoint the live payload is at most T iterations' worth
            live = sum(n for _, _, n in _live_chunks(log_dir)) * rec_bytes
            assert live <= T * per_iter, (it, live)
            _checkpoint(ghost, ckpt_dir, it)
            gc_logs(log_dir, ckpt_dir, it)
            assert all(mx >= it for _, mx, _ in _live_chunks(log_dir)), it
        ghost.run_iteration(cuts=CUTS, senders=loggers)
    assert missing == 0 and replays == POINTS
    for lg in loggers.values():
        lg.close()
