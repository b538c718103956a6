"""Load tests/golden/*.json fixtures into synth.Problem objects."""
import json
import os

import numpy as np

from synth.problem import CrossEdge, Edge, Problem, SegmentType, Transition

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def problem_from(d) -> Problem:
    types = []
    for t in d["types"]:
        types.append(SegmentType(
            radix=np.array(t["radix"], np.int32),
            comp_ns=np.array(t["comp"], np.uint32),
            comm_ns=None if t["comm"] is None else np.array(t["comm"], np.uint32),
            edges=[Edge(a, b, np.array(tab, np.uint32)) for a, b, tab in t["edges"]],
            out_block=t["out_block"],
            mem=None if t.get("mem") is None else np.array(t["mem"], np.uint32)))
    trs = [Transition(x["pred"], x["type"], [CrossEdge(j, np.array(tab, np.uint32))
                                             for j, tab in x["in"]]) for x in d["transitions"]]
    return Problem((1,), types, trs, np.array(d["instances"], np.int32), "golden")
