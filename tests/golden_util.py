"""Loaders for tests/golden/golden.json (made by tests/golden/make_golden.py)."""
import json
import os
import struct
from functools import lru_cache

import numpy as np

from paper_2301_04285_b200.graph import (AxisSlice, ClusterTopology, ComputationGraph, GraphEdge,
                                         OperatorAxis, OperatorNode, TensorSpec)

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")


@lru_cache(maxsize=1)
def golden():
    with open(PATH) as fh:
        return json.load(fh)


def unhex(v):
    if isinstance(v, list):
        return np.array([struct.unpack("<d", bytes.fromhex(x))[0] for x in v], dtype=np.float64)
    return struct.unpack("<d", bytes.fromhex(v))[0]


def graph_of(j):
    ops = []
    for o in j["operators"]:
        ops.append(OperatorNode(
            o["id"], o["kind"], [TensorSpec(t["name"], list(t["shape"]), t["element_size"]) for t in o["inputs"]],
            [TensorSpec(t["name"], list(t["shape"]), t["element_size"]) for t in o["outputs"]],
            [OperatorAxis(a["name"], [AxisSlice(s["tensor"], s["dim"]) for s in a["slices"]]) for a in o["axes"]]))
    return ComputationGraph(ops, [GraphEdge(e["from_"], e["to"], e["tensor"]) for e in j["edges"]])


def topo_of(t):
    return ClusterTopology(t["node_count"], t["local_device_num"], t["intra_bandwidth"], t["inter_bandwidth"],
                           t["device_memory"])


def bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)
