"""Seeded synthetic inputs shared by the oracle and the CUDA path (inputs only)."""
from .problem import (INF32, INF64, NOIDX, CrossEdge, Edge, Problem,  # noqa: F401
                      SegmentType, Transition)
from .generators import (CONFIGS, CONFIG_NAMES, global_plan_count,  # noqa: F401
                         hash_stream, make_config, tiny_random)
