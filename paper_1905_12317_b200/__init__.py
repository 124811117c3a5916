"""B200-native FTK alignment hot path (arXiv:1905.12317): C-ABI library libftk.so + thin binding.

The product path never imports oracle/ (test infrastructure) and has no CPU fallback: if libftk.so
is missing, importing the binding's entry points raises."""
from .api import (ENGINE_SIMT, ENGINE_TC, BEST_DTYPE, FTKError, FTKPlan, best_to_numpy,  # noqa: F401
                  distributed_align, distributed_align_marginal, gather_and_merge, gather_marginal,
                  merge_bests, radial_rule, shard_range, NcclComm)
from ._ffi import LIB_PATH, lib  # noqa: F401
