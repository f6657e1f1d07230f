"""B200-native recovery hot path of Swift (arXiv 2302.06173).

Importing this package loads ``librewind_b200.so`` (built by
``__graft_entry__.build()``) and fails loudly if it is absent.
"""
from ._lib import (ADAM, ADAMW, AMSGRAD, LAMB, SGD, SGDM, RwError)  # noqa: F401
from .optim import (DeviceState, OptimizerHyper, derive_seed, flat_layout,  # noqa: F401
                    invertibility_check, optimizer_from_name, ordered_sum, seeded_fill_)
