"""ctypes binding of the C ABI in include/rewind_b200.h.

The shared library is built in-tree (``paper_2302_06173_b200/librewind_b200.so``)
by ``__graft_entry__.build()``.  There is no fallback: if the library is
missing, importing the package raises, so no product path can silently run on
the CPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "librewind_b200.so"

# 1 + rewind::Err (errors.hpp:11-33), plus B200-side codes.
ERR_NAMES = [
    "OK", "InvalidShape", "ShapeMismatch", "EmptyInput", "NumericalError",
    "NonInvertibleHyper", "NotInvertible", "NothingToUndo", "AlreadyUpdated",
    "MissingActivation", "ChannelBroken", "InvalidInjection", "NotFailed",
    "StorageError", "MissingLogData", "CorruptLog", "NoCheckpoint", "NoReplica",
    "InvalidConfig", "TooLarge",
]
RW_CUDA_ERROR = 100
RW_INVALID_ARGUMENT = 101

SGD, SGDM, ADAM, ADAMW, LAMB, AMSGRAD = range(6)
F32, F64 = 0, 1
INVERTIBLE, INVERTIBLE_WITH_SAVED_SCALARS, NOT_INVERTIBLE = range(3)
ACT_NONE, ACT_UNDO, ACT_REDO = range(3)
POLICY_UNDO, POLICY_MIN_COST = range(2)
STRATEGY_NONE, STRATEGY_UNDO, STRATEGY_REDO, STRATEGY_GLOBAL_ROLLBACK = range(4)
STRATEGY_NAMES = {0: "None", 1: "Undo", 2: "Redo", 3: "GlobalRollback"}


class RwError(RuntimeError):
    """Mirror of ``rewind::Error`` (errors.hpp:37-44): carries the Err code."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = status - 1 if 1 <= status <= 19 else None
        self.name = ERR_NAMES[status] if 0 <= status < len(ERR_NAMES) else (
            "CudaError" if status == RW_CUDA_ERROR else "InvalidArgument")
        super().__init__(message or self.name)


class rw_hyper(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("require_invertible", C.c_int32),
        ("lr", C.c_double), ("weight_decay", C.c_double), ("momentum", C.c_double),
        ("dampening", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
        ("eps", C.c_double),
        ("lr_table_from", C.POINTER(C.c_uint64)), ("lr_table_value", C.POINTER(C.c_double)),
        ("lr_table_len", C.c_uint32), ("_pad", C.c_uint32),
    ]


class rw_group(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("len", C.c_uint64), ("t", C.c_uint64),
                ("updated", C.c_uint32), ("flags", C.c_uint32)]


class rw_resolve_summary(C.Structure):
    _fields_ = [("t_min", C.c_uint64), ("t_max", C.c_uint64), ("undo_elems", C.c_uint64),
                ("redo_elems", C.c_uint64), ("redo_blocked", C.c_uint64),
                ("undo_blocked", C.c_uint64)]


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: run __graft_entry__.build() (the B200 path has no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
    vp, u32, u64, i32, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32, C.c_double
    P = C.POINTER
    sig = {
        "rw_abi_version": (C.c_int, []),
        "rw_last_error_message": (C.c_char_p, []),
        "rw_status_name": (C.c_char_p, [C.c_int]),
        "rw_device_count": (C.c_int, []),
        "rw_invertibility_check": (C.c_int, [i32]),
        "rw_hyper_validate": (C.c_int, [P(rw_hyper)]),
        "rw_lr_at": (C.c_int, [P(rw_hyper), u64, P(dbl)]),
        "rw_state_create": (C.c_int, [P(vp), i32, vp, vp, vp, vp, vp, u64, P(rw_group), u32, i32]),
        "rw_state_create_host": (C.c_int, [P(vp), i32, u64, P(rw_group), u32, i32]),
        "rw_state_destroy": (None, [vp]),
        "rw_state_num_groups": (u32, [vp]),
        "rw_state_read_groups": (C.c_int, [vp, P(rw_group), vp]),
        "rw_state_write_groups": (C.c_int, [vp, P(rw_group), vp]),
        "rw_state_check": (C.c_int, [vp, vp]),
        "rw_clear_updated": (C.c_int, [vp, P(u32), u32, vp]),
        "rw_state_ptr": (vp, [vp, C.c_int]),
        "rw_optimizer_step": (C.c_int, [vp, P(rw_hyper), P(u32), u32, vp, u32, vp]),
        "rw_optimizer_undo": (C.c_int, [vp, P(rw_hyper), P(u32), u32, vp]),
        "rw_resolve_summarize": (C.c_int, [P(rw_group), u32, P(C.c_uint8), P(rw_hyper), u64,
                                           P(rw_resolve_summary)]),
        "rw_resolve_plan": (C.c_int, [P(rw_resolve_summary), i32, P(rw_group), u32,
                                      P(C.c_uint8), P(u64), P(i32)]),
        "rw_seeded_fill": (C.c_int, [i32, vp, u64, u64, u64, vp]),
        "rw_derive_seed": (u64, [u64, P(u64), u32]),
        "rw_ordered_sum": (C.c_int, [i32, P(vp), u32, u64, vp, vp]),
        "rw_bubble_ratio": (C.c_int, [i32, i32, P(C.c_int64), P(C.c_int64)]),
        "rw_group_machines": (C.c_int, [u32, P(dbl), P(dbl), dbl, dbl, dbl, i32, P(u32),
                                        P(u32), P(dbl), P(dbl)]),
        "rw_recovery_time_estimate": (C.c_int, [u32, P(dbl), P(dbl), dbl, i32, P(u32), dbl,
                                                P(dbl)]),
        "rw_logging_worthwhile": (C.c_int, [dbl, dbl, i32, i32, dbl, P(i32), P(dbl), P(dbl)]),
        "rw_ipc_export": (C.c_int, [vp, vp, P(u64)]),
        "rw_ipc_import": (C.c_int, [vp, P(vp)]),
        "rw_ipc_close": (C.c_int, [vp]),
        "rw_undo_and_push": (C.c_int, [vp, P(rw_hyper), P(u32), u32, vp, vp, vp, vp, vp]),
        "rw_host_block_step": (C.c_int, [i32, vp, vp, vp, vp, vp, u64, P(u64), P(u32), vp,
                                         P(rw_hyper)]),
        "rw_host_block_undo": (C.c_int, [i32, vp, vp, vp, vp, u64, P(u64), P(u32), P(rw_hyper)]),
        "rw_host_block_lamb_step": (C.c_int, [i32, vp, vp, vp, vp, u64, P(u64), P(u32), vp,
                                              P(rw_hyper), P(dbl)]),
        "rw_host_block_lamb_undo": (C.c_int, [i32, vp, vp, vp, vp, u64, P(u64), P(u32),
                                              P(rw_hyper), u32, dbl]),
        "rw_optimizer_undo_host": (C.c_int, [vp, P(rw_hyper), P(u32), u32, vp, vp, vp, vp, vp, vp, vp, u64,
                                             vp]),
        "rw_copy_async": (C.c_int, [P(vp), P(vp), P(u64), u32, vp]),
        "rw_stream_write_u64": (C.c_int, [vp, vp, u64]),
        "rw_stream_wait_u64": (C.c_int, [vp, vp, u64]),
        "rw_state_saved_scalars": (C.c_int, [vp, u32, P(dbl), u32, P(u32), vp]),
        "rw_state_set_saved_scalars": (C.c_int, [vp, u32, P(dbl), u32, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()
if LIB.rw_abi_version() != 1:
    raise ImportError("librewind_b200.so ABI version mismatch")


def check(status: int) -> None:
    """Raise RwError (the rewind::Error mirror) for a non-zero status."""
    if status != 0:
        msg = LIB.rw_last_error_message()
        raise RwError(status, msg.decode() if msg else "")


def declared_functions() -> list[str]:
    """Names of every function declared in include/rewind_b200.h."""
    import re
    hdr = (_HERE.parent / "include" / "rewind_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][A-Za-z0-9_ \*]*?)\b(rw_[a-z0-9_]+)\s*\(",
                                 hdr, flags=re.M)))


def library_exports() -> set[str]:
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def default_stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


os.environ.setdefault("REWIND_B200_LIB", str(LIB_PATH))
