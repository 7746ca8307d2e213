"""Dump a workload's flattened graph + topology for the host-analysis probe."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2301_04285_b200 import graph as G, models as M

g, t = M.cfg4()
f = G.flatten(g)
keys = ["op_id", "op_tensor_begin", "op_num_inputs", "op_axis_begin", "tensor_name", "tensor_shape_begin",
        "shape", "tensor_element_size", "axis_slice_begin", "slice_tensor", "slice_dim", "edge_from", "edge_to",
        "edge_tensor"]
with open(sys.argv[1], "wb") as fh:
    np.array([f.num_ops, f.num_edges, t.node_count, t.local_device_num], np.int64).tofile(fh)
    np.array([t.intra_bandwidth, t.inter_bandwidth, t.device_memory], np.float64).tofile(fh)
    for k in keys:
        a = getattr(f, k)
        np.array([a.size], np.int64).tofile(fh)
        a.tofile(fh)
