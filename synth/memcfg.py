"""Memory-constrained workloads: a config's problem plus
a quantum and a device memory limit.  Input sizing only -- no arithmetic of
the method: the limit is placed a fraction of the way between the chain's
smallest and largest possible memory (sums of per-block min / max m_j[s],
App. C memory model in KiB) so that it binds, and the quantum splits the
limit into `levels` quanta (Qmax = levels)."""
from __future__ import annotations

import math

from .generators import make_config


# quanta per limit: enough that the per-block ceilings of a deep chain still
# leave room between the smallest and largest quantised plan memory
LEVELS = {"C1": 64, "C2": 256, "C3": 256, "C4": 512, "C5": 1024}


def mem_workload(cfg: str = "C3", seed: int = 0, dist: str = "shaped", levels: int = 0,
                 frac: float = 0.35):
    levels = levels or LEVELS.get(cfg, 256)
    p = make_config(cfg, seed, dist)
    lo = hi = 0
    for t in p.instances:
        ty = p.types[p.transitions[int(t)].type]
        for j in range(len(ty.radix)):
            m = ty.mem_of(j)
            lo += int(m.min())
            hi += int(m.max())
    limit = int(lo + frac * (hi - lo))
    quantum = max(1, math.ceil(limit / levels))
    return p, quantum, limit
