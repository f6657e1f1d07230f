"""Checkpoint store + log GC host logic, no GPU:
host blobs only, driven through the C ABI.  The SPEC examples:
  * load a nonexistent manifest -> NoCheckpoint
  * crash mid-write -> latest valid manifest is the prior one
  * ckpt at 100 -> chunks covering 0..99 deleted, 100+ retained; gc twice idempotent
"""
import ctypes as C
import os
import struct

import numpy as np
import pytest

from paper_2302_06173_b200 import RwError
from paper_2302_06173_b200._lib import LIB, check
from paper_2302_06173_b200.checkpoint import NO_CRASH, gc_logs, latest_checkpoint, rw_blob


_KEEP = []  # the arrays behind the raw pointers must outlive the calls


def _blobs(arrs: dict):
    _KEEP.append(arrs)
    bl = [rw_blob(k.encode(), C.c_void_p(a.ctypes.data), a.nbytes, 1, 0) for k, a in arrs.items()]
    return (rw_blob * len(bl))(*bl), len(bl)


def _write(d, it, worker, arrs, crash=NO_CRASH):
    arr, n = _blobs(arrs)
    return LIB.rw_ckpt_write(str(d).encode(), it, worker, arr, n, crash, None)


def test_write_commit_load_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    w0 = {"s0.x": rng.standard_normal(1000), "s0.m": rng.standard_normal(1000), "meta.json": np.frombuffer(
        b'{"a": 1}', dtype=np.uint8).copy()}
    w1 = {"s0.x": rng.standard_normal(77), "meta.json": np.frombuffer(b"{}", dtype=np.uint8).copy()}
    with pytest.raises(RwError) as e:
        latest_checkpoint(str(tmp_path))
    assert e.value.name == "NoCheckpoint"
    check(_write(tmp_path, 100, 0, w0))
    # worker 1 has not written: the global manifest must not appear
    assert LIB.rw_ckpt_commit(str(tmp_path).encode(), 100, 2) == 13  # StorageError
    with pytest.raises(RwError):
        latest_checkpoint(str(tmp_path))
    check(_write(tmp_path, 100, 1, w1))
    check(LIB.rw_ckpt_commit(str(tmp_path).encode(), 100, 2))
    assert latest_checkpoint(str(tmp_path)) == 100
    out = {k: np.zeros_like(v) for k, v in w0.items()}
    arr, n = _blobs(out)
    check(LIB.rw_ckpt_load(str(tmp_path).encode(), 100, 0, arr, n, None))
    for k in w0:
        assert np.array_equal(out[k], w0[k])
    out1 = {"s0.x": np.zeros(77)}
    arr, n = _blobs(out1)
    check(LIB.rw_ckpt_load(str(tmp_path).encode(), 100, 1, arr, n, None))
    assert np.array_equal(out1["s0.x"], w1["s0.x"])
    # size mismatch -> ShapeMismatch, before any byte moves
    bad = {"s0.x": np.zeros(999)}
    arr, n = _blobs(bad)
    assert LIB.rw_ckpt_load(str(tmp_path).encode(), 100, 0, arr, n, None) == 2
    # unknown blob / worker / iteration
    arr, n = _blobs({"nope": np.zeros(3)})
    assert LIB.rw_ckpt_load(str(tmp_path).encode(), 100, 0, arr, n, None) == 13
    arr, n = _blobs({"s0.x": np.zeros(1000)})
    assert LIB.rw_ckpt_load(str(tmp_path).encode(), 100, 2, arr, n, None) == 16  # NoCheckpoint
    assert LIB.rw_ckpt_load(str(tmp_path).encode(), 101, 0, arr, n, None) == 16


def test_torn_write_keeps_previous_manifest(tmp_path):
    a = {"s0.x": np.arange(10.0), "s0.m": np.arange(10.0) * 2, "meta.json": np.zeros(4, np.uint8)}
    check(_write(tmp_path, 100, 0, a))
    check(LIB.rw_ckpt_commit(str(tmp_path).encode(), 100, 1))
    b = {k: v + 1 for k, v in a.items()}
    st = _write(tmp_path, 150, 0, b, crash=1)  # dies after the first blob
    assert st == 13
    assert LIB.rw_ckpt_commit(str(tmp_path).encode(), 150, 1) == 13  # no worker manifest
    assert latest_checkpoint(str(tmp_path)) == 100
    out = {"s0.x": np.zeros(10)}
    arr, n = _blobs(out)
    check(LIB.rw_ckpt_load(str(tmp_path).encode(), 100, 0, arr, n, None))
    assert np.array_equal(out["s0.x"], a["s0.x"])
    assert LIB.rw_ckpt_load(str(tmp_path).encode(), 150, 0, arr, n, None) == 16


def test_corrupt_blob_is_detected(tmp_path):
    a = {"s0.x": np.linspace(0, 1, 4096)}
    check(_write(tmp_path, 7, 0, a))
    check(LIB.rw_ckpt_commit(str(tmp_path).encode(), 7, 1))
    p = tmp_path / "ck_0000000000000007" / "w00000" / "s0.x.bin"
    raw = bytearray(p.read_bytes())
    raw[100] ^= 0x40
    p.write_bytes(bytes(raw))
    arr, n = _blobs({"s0.x": np.zeros(4096)})
    assert LIB.rw_ckpt_load(str(tmp_path).encode(), 7, 0, arr, n, None) == 13
    assert b"checksum" in LIB.rw_last_error_message()
    # truncated blob
    p.write_bytes(bytes(raw[:-8]))
    assert LIB.rw_ckpt_load(str(tmp_path).encode(), 7, 0, arr, n, None) == 13


def _chunk(path, machine, records):
    """An SWFT chunk file in the documented format."""
    out = bytearray(b"SWFT" + struct.pack("<HI", 1, machine))
    for it, mb, payload in records:
        shape = [len(payload)]
        body = struct.pack("<IIQIBBBB", 0, 1, it, mb, 0, 2, len(shape), 0)
        body += b"".join(struct.pack("<Q", s) for s in shape) + struct.pack("<Q", len(payload)) + payload
        body += struct.pack("<I", 0)
        out += struct.pack("<I", len(body)) + body
    with open(path, "wb") as f:
        f.write(out)


def test_gc_logs(tmp_path):
    logs, ck = tmp_path / "logs", tmp_path / "ck"
    logs.mkdir()
    for c in range(6):  # chunk c covers iterations 20c .. 20c+19
        _chunk(logs / f"m0001_{c:08d}.swft", 1,
               [(20 * c + k, k % 4, bytes([k]) * 16) for k in range(0, 20, 5)])
    (logs / "m0001_00000006.swft.tmp").write_bytes(b"partial")
    with pytest.raises(RwError) as e:  # pre: the checkpoint is committed
        gc_logs(str(logs), str(ck), 100)
    assert e.value.name == "NoCheckpoint"
    a = {"meta.json": np.zeros(1, np.uint8)}
    check(_write(ck, 100, 0, a))
    check(LIB.rw_ckpt_commit(str(ck).encode(), 100, 1))
    assert gc_logs(str(logs), str(ck), 100) == 5  # chunks 0..4 (max it 99) go; chunk 5 (100+) stays
    left = sorted(os.listdir(logs))
    assert left == ["m0001_00000005.swft", "m0001_00000006.swft.tmp"]
    assert gc_logs(str(logs), str(ck), 100) == 0  # idempotent
