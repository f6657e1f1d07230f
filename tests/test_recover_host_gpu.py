"""The C++ recovery host (csrc/recovery_host.cpp, csrc/replay_host.cpp) driven
by a multi-process C++ program through the C ABI only (tests/cpp/
recover_host_test.cpp): replica recovery, parallel replay and NCCL-native
failure detection + communicator repair, one process per GPU.  Needs >= 2
GPUs (NCCL refuses two ranks on one device)."""
import os
import subprocess

import pytest
import torch

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "recover_host_test")
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
need2 = pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs (one NCCL rank per device)")


def _run(*args, timeout=600):
    try:
        out = subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    except subprocess.TimeoutExpired as e:  # show how far every rank got
        def tail(b):
            return (b.decode(errors="replace") if isinstance(b, bytes) else (b or ""))[-4000:]
        raise AssertionError(f"timed out after {timeout} s\n{tail(e.stdout)}\n{tail(e.stderr)}") from None
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "PASS" in out.stdout, out.stdout[-4000:]
    return out.stdout


@need2
@pytest.mark.parametrize("mode", ["nccl", "chain"])
@pytest.mark.parametrize("n", sorted({2, min(NGPU, 4)}))
def test_cpp_replication(n, mode):
    """Pipelined undo + NCCL broadcasts, or the copy-engine chain
    (RW_RECOVER_CHAIN): every replica's CRC equals the survivor's."""
    print(_run("replication", n, *(["chain"] if mode == "chain" else [])))


@need2
def test_cpp_parallel_replay():
    print(_run("replay", 2))


@need2
def test_cpp_failure_detection_shrink_and_join():
    print(_run("failure", min(NGPU, 3)))
