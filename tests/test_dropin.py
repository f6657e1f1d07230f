"""The C++ header-only drop-in (include/rewind_b200.hpp) driven with the
reference's own ParamBlock/Tensor/OptimizerHyper objects, compared with the
reference library bit for bit (tests/cpp/dropin_test.cpp)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "dropin_test"


def _run(*args):
    if not BIN.exists():
        pytest.fail(f"{BIN} not built: run __graft_entry__.build()")
    r = subprocess.run([str(BIN), *args], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout


def test_dropin_guards_cpu():
    _run("--cpu")


@pytest.mark.gpu
def test_dropin_bitexact_vs_reference_gpu():
    _run()


@pytest.mark.gpu
def test_cpp_host_resolve_and_undo_gpu():
    """A C++ host (no Python in the loop) repairs a torn fp64 Adam update
    through the C ABI (read markers, resolve, undo) and matches the
    reference's optimizer_step / optimizer_undo bit for bit
    (tests/cpp/resolve_undo_test.cpp)."""
    b = BIN.parent / "resolve_undo_test"
    if not b.exists():
        pytest.fail(f"{b} not built: run __graft_entry__.build()")
    r = subprocess.run([str(b)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "0 failure(s)" in r.stdout, r.stdout + r.stderr
