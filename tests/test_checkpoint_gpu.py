"""Checkpoint store on the device path: device blobs through
the pinned D2H/H2D pipeline with GPU CRC32, and the SPEC example
"checkpoint at c, load, rerun -> trajectory bit-identical to the
uninterrupted run" on the replay path (load from disk + replay from log
files == ghost run, bit for bit)."""
import numpy as np
import pytest
import torch

from paper_2302_06173_b200 import ADAM, LAMB, DeviceState, OptimizerHyper, RwError, seeded_fill_
from paper_2302_06173_b200.checkpoint import gc_logs, latest_checkpoint, load_checkpoint, write_checkpoint

pytestmark = pytest.mark.gpu


def _adam_state(sizes, seed, kind=ADAM):
    st = DeviceState(sizes, kind=kind)
    seeded_fill_(st.x, seed)
    seeded_fill_(st.g, seed + 1)
    seeded_fill_(st.m, seed + 2)
    seeded_fill_(st.v, seed + 3)
    st.v.abs_()
    return st


def test_device_roundtrip_bitexact(tmp_path):
    # > one 64 MiB staging chunk per blob so the ring wraps
    sizes = [20_000_000, 3, 4_000_001]
    a = _adam_state(sizes, 11)
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    a.step(h, stop_after=2)  # torn markers travel with the state
    b = _adam_state([5000, 7], 3, kind=LAMB)
    hl = OptimizerHyper(kind=LAMB, lr=1e-3, weight_decay=0.01)
    b.step(hl)
    write_checkpoint([a, b], str(tmp_path), 40, include_grad=True, extra={"rng": [1, 2, 3]})
    assert latest_checkpoint(str(tmp_path)) == 40
    ra = DeviceState(sizes, kind=ADAM)
    rb = DeviceState([5000, 7], kind=LAMB)
    it, extra = load_checkpoint([ra, rb], str(tmp_path))
    assert it == 40 and extra == {"rng": [1, 2, 3]}
    for src, dst in ((a, ra), (b, rb)):
        for n in ("x", "g", "m", "v"):
            assert torch.equal(getattr(src, n), getattr(dst, n)), n
        assert src.markers() == dst.markers()
    assert [rb.saved_scalars(i) for i in range(2)] == [b.saved_scalars(i) for i in range(2)]
    # the restored LAMB state undoes exactly like the original
    b.undo(hl)
    rb.undo(hl)
    assert torch.equal(b.x, rb.x) and torch.equal(b.m, rb.m) and torch.equal(b.v, rb.v)
    # layout mismatch -> ShapeMismatch
    with pytest.raises(RwError) as e:
        load_checkpoint([DeviceState([5, 5], kind=ADAM), rb], str(tmp_path))
    assert e.value.name == "ShapeMismatch"
    # device-side CRC catches a flipped byte deep inside a multi-chunk blob
    parts = sorted((tmp_path / "ck_0000000000000040" / "w00000").glob("s0.m.bin.*"))
    assert len(parts) == 3  # 96 MB blob -> three 32 MiB parts written in parallel
    with open(parts[-1], "r+b") as f:
        f.seek(6 << 20)
        c = f.read(1)
        f.seek(6 << 20)
        f.write(bytes([c[0] ^ 1]))
    with pytest.raises(RwError) as e:
        load_checkpoint([ra, rb], str(tmp_path))
    assert e.value.name == "StorageError" and "checksum" in str(e.value)


def test_checkpoint_feeds_replay_from_files(tmp_path):
    """Ghost run of a 3-stage pipeline logging stage 1's boundary tensors to
    SWFT files and checkpointing stage 1 to disk at iteration 2; a replacement
    loads the checkpoint from disk, replays iterations 2..4 from the files and
    must equal the ghost bit for bit.  gc_logs then drops the pre-checkpoint
    chunks only, and replay from the surviving chunks still matches."""
    from paper_2302_06173_b200 import logstore
    from paper_2302_06173_b200.replay import Pipeline, Stage, replay_group
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    ghost = Pipeline(p=3, dim=64, hidden=128, layers=2, rows=128, micro_batches=4, seed=5, kind=ADAM, hyper=h)
    logs, ck = tmp_path / "logs", tmp_path / "ck"
    lg = logstore.Logger(str(logs), machine=1, chunk_records=8, pinned_bytes=8 << 20)
    for it in range(5):
        if it == 2:
            lg.flush()  # chunk boundary at the checkpoint (records of 0..1 in earlier chunks)
            write_checkpoint(ghost.stages[1].state, str(ck), 2, extra={"iteration": 2})
        ghost.run_iteration(log_group=(1, 1), log=lg)
    lg.flush()
    lg.close()
    assert gc_logs(str(logs), str(ck), 2) >= 1
    rep = Stage(1, 64, 128, 64, 2, 5, ADAM)
    it, extra = load_checkpoint(rep.state, str(ck))
    rep.refresh_shadows()
    assert it == 2 and extra["iteration"] == 2
    loaded = logstore.load_log_dir(str(logs))
    assert min(k[0] for k in loaded.acts) == 2
    replay_group([rep], loaded, 2, 5, 128, 4, 5, h, first=False, last=False, dim=64)
    g = ghost.stages[1].state
    assert torch.equal(rep.state.x, g.x) and torch.equal(rep.state.m, g.m) and torch.equal(rep.state.v, g.v)
    assert rep.state.markers() == g.markers()
    assert np.all(np.array([t for t, _ in g.markers()]) == 5)
