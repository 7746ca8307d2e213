"""price_assignment on the device (tp_plan_price_assignments) against the
reference's summation (aux_graph.hpp:326-348) restated over the oracle's
tensors: topological order, a source's virtual edge first, then every edge
whose `to` id equals the operator's id, ascending -- bit-exact in both cost
modes and for the memory sum."""
import random

import numpy as np
import pytest

from oracle import bindings as B
from paper_2301_04285_b200 import engine, fuzz, graph as G, models as M

pytestmark = pytest.mark.gpu


def ref_price(f, ref, asg):
    cost = vol = mem = 0.0
    nb, eb = ref.node_base, ref.edge_base
    for op in ref.topo_order:
        op = int(op)
        node = int(nb[op]) + int(asg[op])
        if ref.in_degree[op] == 0:
            cost += float(ref.node_intra_cost_s[node])
            vol += float(ref.node_intra_volume_bytes[node])
            mem += float(ref.node_memory_bytes[node])
        for e in range(f.num_edges):
            if f.edge_to[e] != f.op_id[op]:
                continue
            u, w = int(ref.edge_from_op[e]), int(ref.edge_to_op[e])
            a = int(eb[e]) + int(asg[u]) * int(nb[w + 1] - nb[w]) + int(asg[op])
            cost += float(ref.edge_cost_s[a])
            vol += float(ref.edge_volume_bytes[a])
            mem += float(ref.edge_memory_bytes[a])
    return cost, vol, mem


def check(g, t, k, seed):
    import torch
    f = G.flatten(g)
    ref = B.oracle_build(f, t)
    assert ref.status == 0
    plan = engine.Plan(f, t, device=0)
    ne, nn = plan.sizes["num_aux_edges"], plan.sizes["num_aux_nodes"]
    dev = torch.device("cuda", 0)
    outs = {kk: torch.empty(max(ne, 1), dtype=torch.float64, device=dev)
            for kk in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")}
    outs.update({kk: torch.empty(max(nn, 1), dtype=torch.float64, device=dev)
                 for kk in ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes")})
    s = torch.cuda.current_stream().cuda_stream
    plan.execute(engine.device_cost_struct(outs), stream=s)
    plan.check_errors()
    rng = random.Random(seed)
    S = [int(ref.node_base[i + 1] - ref.node_base[i]) for i in range(f.num_ops)]
    asg = np.array([[rng.randrange(S[i]) for i in range(f.num_ops)] for _ in range(k)], np.int32)
    c, v, m = plan.price_assignments(outs, torch.from_numpy(asg).to(dev), stream=s)
    torch.cuda.synchronize()
    c, v, m = c.cpu().numpy(), v.cpu().numpy(), m.cpu().numpy()
    for j in range(k):
        rc, rv, rm = ref_price(f, ref, asg[j])
        assert np.float64(rc).view(np.uint64) == c[j:j + 1].view(np.uint64)[0], (j, rc, c[j])
        assert np.float64(rv).view(np.uint64) == v[j:j + 1].view(np.uint64)[0], (j, rv, v[j])
        assert np.float64(rm).view(np.uint64) == m[j:j + 1].view(np.uint64)[0], (j, rm, m[j])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_price_assignments_configs(cfg):
    g, t = getattr(M, cfg)()
    check(g, t, 64, 3)


def test_price_assignments_gpt_chain():
    g, t = M.cfg3(2)
    check(g, t, 16, 4)


def test_price_assignments_random_graphs():
    rng = random.Random(11)
    done = 0
    for i in range(120):
        g, t = fuzz.random_graph(rng, odd_extents=False)
        f = G.flatten(g)
        if B.oracle_build(f, t).status != 0:
            continue
        check(g, t, 8, i)
        done += 1
    assert done >= 10
