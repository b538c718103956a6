"""B200-native CFP plan-search hot path (arXiv 2504.00598).

The product is libcfp.so (include/cfp.h): sm_100a kernels for exhaustive
strategy-combination evaluation, the min-plus segment chain and the plan
backtrack.  `cfp` is its thin ctypes binding.
"""
from . import cfp  # noqa: F401
from .cfp import CfpError, Context, Plan, Prepared  # noqa: F401

__all__ = ["cfp", "CfpError", "Context", "Plan", "Prepared"]
