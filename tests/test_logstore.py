"""Log store: GPU CRC32 vs the reference crc32 (wire.cpp:31-38),
the SWFT chunk format, the async logger, and replay from log files."""
import glob
import os
import struct

import numpy as np
import pytest
import torch

from paper_2302_06173_b200 import RwError
from paper_2302_06173_b200 import logstore


def _write_swft(path, machine, records):
    """Test-side writer of the documented format (DESIGN.md §log format)."""
    with open(path, "wb") as f:
        f.write(b"SWFT" + struct.pack("<HI", 1, machine))
        for (sender, receiver, it, mb, direction, dtype, shape, payload, crc) in records:
            body = struct.pack("<IIQIBBBB", sender, receiver, it, mb, direction, dtype, len(shape), 0)
            body += b"".join(struct.pack("<Q", s) for s in shape)
            body += struct.pack("<Q", len(payload)) + payload + struct.pack("<I", crc)
            f.write(struct.pack("<I", len(body)) + body)


def test_reader_parses_format_cpu(tmp_path, ref):
    payload = np.arange(24, dtype=np.float32).tobytes()
    p = str(tmp_path / "m0003_00000000.swft")
    _write_swft(p, 3, [(2, 3, 7, 1, 0, 0, (2, 3, 4), payload, ref.crc32(payload)),
                       (4, 3, 7, 1, 1, 0, (24,), payload, 0xDEADBEEF)])
    recs = list(logstore.read_chunk(p))
    assert len(recs) == 2
    r, pay = recs[0]
    assert (r.sender, r.receiver, r.iteration, r.mb, r.direction, r.ndim) == (2, 3, 7, 1, 0, 3)
    assert [r.shape[i] for i in range(3)] == [2, 3, 4]
    assert bytes(pay.numpy()) == payload and r.crc32 == ref.crc32(payload)
    assert recs[1][0].crc32 == 0xDEADBEEF


def test_reader_errors_cpu(tmp_path):
    with pytest.raises(RwError) as e:
        list(logstore.read_chunk(str(tmp_path / "nope.swft")))
    assert e.value.name == "MissingLogData"
    bad = tmp_path / "bad.swft"
    bad.write_bytes(b"NOPE\x01\x00\x00\x00\x00\x00")
    with pytest.raises(RwError) as e:
        list(logstore.read_chunk(str(bad)))
    assert e.value.name == "CorruptLog"
    p = str(tmp_path / "trunc.swft")
    _write_swft(p, 0, [(0, 1, 0, 0, 0, 0, (4,), b"\0" * 16, 0)])
    data = open(p, "rb").read()
    open(p, "wb").write(data[:-7])  # truncated payload/crc
    with pytest.raises(RwError) as e:
        list(logstore.read_chunk(p))
    assert e.value.name == "CorruptLog"


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 9, 255, 256, 257, 65535, 65536, 65537, 3 * 65536 + 1000, 10_000_003])
def test_crc32_device_matches_reference(ref, n):
    rng = np.random.default_rng(n)
    data = b"123456789" if n == 9 else rng.integers(0, 256, n, dtype=np.uint8).tobytes()
    t = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda() if n else torch.empty(0, dtype=torch.uint8,
                                                                                          device="cuda")
    assert logstore.crc32_device(t) == ref.crc32(data)
    if n == 9:
        assert logstore.crc32_device(t) == 0xCBF43926


@pytest.mark.gpu
@pytest.mark.parametrize("offset", [1, 4, 16, 32])
@pytest.mark.parametrize("n", [65536 * 5 + 7, 1_000_003])
def test_crc32_device_any_alignment(ref, offset, n):
    """The chunk kernel reads 32-byte aligned pieces with 256-bit loads and
    takes a byte-load variant for any other address: same CRC either way."""
    rng = np.random.default_rng(offset)
    data = rng.integers(0, 256, n + offset, dtype=np.uint8).tobytes()
    t = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()[offset:]
    assert logstore.crc32_device(t) == ref.crc32(data[offset:])


@pytest.mark.gpu
def test_logger_roundtrip_and_replay_from_files(tmp_path):
    from paper_2302_06173_b200 import ADAM, OptimizerHyper
    from paper_2302_06173_b200.replay import BoundaryLog, Pipeline, Stage, replay_group
    h = OptimizerHyper(kind=ADAM, lr=1e-3, weight_decay=0.01)
    mk = lambda: Pipeline(p=3, dim=64, hidden=128, layers=2, rows=128, micro_batches=4, seed=5,  # noqa: E731
                          kind=ADAM, hyper=h)
    ghost_mem, ghost_file = mk(), mk()
    mem = BoundaryLog()
    lg = logstore.Logger(str(tmp_path), machine=1, chunk_records=5, pinned_bytes=8 << 20)
    for it in range(3):
        if it == 1:
            snap = ghost_file.stages[1].snapshot()
        ghost_mem.run_iteration(log_group=(1, 1), log=mem)
        ghost_file.run_iteration(log_group=(1, 1), log=lg)
    n = lg.flush()
    lg.close()
    assert n == 3 * 4 * 2
    files = sorted(glob.glob(str(tmp_path / "*.swft")))
    assert not glob.glob(str(tmp_path / "*.tmp"))  # every chunk committed (renamed)
    per_file = [len(list(logstore.read_chunk(f))) for f in files]  # writer lanes: one open chunk each
    assert sum(per_file) == 24 and max(per_file) <= 5
    loaded = logstore.load_log_dir(str(tmp_path))
    assert set(loaded.acts) == set(mem.acts) and set(loaded.grads) == set(mem.grads)
    for k in mem.acts:
        assert torch.equal(loaded.acts[k], mem.acts[k])
        assert torch.equal(loaded.grads[k], mem.grads[k])
    rep = Stage(1, 64, 128, 64, 2, 5, ADAM)
    rep.restore(snap)
    replay_group([rep], loaded, 1, 3, 128, 4, 5, h, first=False, last=False, dim=64)
    assert torch.equal(rep.state.x, ghost_file.stages[1].state.x)
    assert torch.equal(rep.state.v, ghost_file.stages[1].state.v)
    # corrupt one payload byte -> CorruptLog at load time
    with open(files[2], "r+b") as f:
        f.seek(200)
        b = f.read(1)
        f.seek(200)
        f.write(bytes([b[0] ^ 0xFF]))
    with pytest.raises(RwError) as e:
        logstore.load_log_dir(str(tmp_path))
    assert e.value.name in ("CorruptLog",)


@pytest.mark.gpu
def test_logger_does_not_block_producer_stream(tmp_path):
    lg = logstore.Logger(str(tmp_path), machine=0, chunk_records=64, pinned_bytes=64 << 20)
    t = torch.randn(4096, 1024, device="cuda").to(torch.bfloat16)
    for i in range(8):
        lg.log_send(t, 0, 1, i, 0, logstore.RW_LOG_ACTIVATION)
    assert lg.flush() == 8
    lg.close()
    recs = [rec for f in sorted(glob.glob(str(tmp_path / "*.swft"))) for rec in logstore.read_chunk(f)]
    assert len(recs) == 8 and all(r.payload_bytes == t.numel() * 2 for r, _ in recs)
    assert sorted(r.iteration for r, _ in recs) == list(range(8))
    assert all(r.crc32 == logstore.crc32_device(t) for r, _ in recs)
