"""B200-native recovery hot path of Swift (arXiv 2302.06173).

The public names below load ``librewind_b200.so`` (built by
``__graft_entry__.build()``) on first use and fail loudly if it is absent.
Pure-host modules (``workloads``) import without touching the library, so the
reference arm of bench.py never maps the product .so.
"""
from __future__ import annotations

import importlib

_LAZY = {
    "_lib": ("ADAM", "ADAMW", "AMSGRAD", "LAMB", "SGD", "SGDM", "RwError"),
    "optim": ("DeviceState", "OptimizerHyper", "derive_seed", "flat_layout", "invertibility_check",
              "optimizer_from_name", "ordered_sum", "seeded_fill_"),
}
_WHERE = {name: mod for mod, names in _LAZY.items() for name in names}
__all__ = sorted(_WHERE)


def __getattr__(name: str):
    mod = _WHERE.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    value = getattr(importlib.import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value
