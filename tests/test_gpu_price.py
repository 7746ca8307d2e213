"""price_assignment on the device (tp_plan_price_assignments) against the
reference's own price_assignment (aux_graph.hpp:326-348, run through
oracle/_ref's ref_price_assignments on the reference's own build): bit-exact
in both cost modes and for the memory sum. The Python restatement of the
summation order (topological order, a source's virtual edge first, then every
edge whose `to` id equals the operator's id, ascending) is pinned to the
reference on CPU (test_restatement_matches_reference)."""
import random

import numpy as np
import pytest

from oracle import bindings as B
from paper_2301_04285_b200 import engine, fuzz, graph as G, models as M



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
    if B.have_reference():  # the reference's own price_assignment
        rc, rv, rm = B.reference_price_assignments(f, t, asg)
    else:
        rc, rv, rm = (np.array(x) for x in zip(*[ref_price(f, ref, asg[j]) for j in range(k)]))
    assert rc.view(np.uint64).tolist() == c.view(np.uint64).tolist()
    assert rv.view(np.uint64).tolist() == v.view(np.uint64).tolist()
    assert rm.view(np.uint64).tolist() == m.view(np.uint64).tolist()


@pytest.mark.skipif(not B.have_reference(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_restatement_matches_reference(cfg):
    """CPU: the summation restated over the oracle's tensors equals the
    reference's price_assignment bit for bit (both modes, memory)."""
    g, t = M.cfg3(2) if cfg == "cfg3" else getattr(M, cfg)()
    f = G.flatten(g)
    ref = B.oracle_build(f, t)
    rng = random.Random(5)
    S = [int(ref.node_base[i + 1] - ref.node_base[i]) for i in range(f.num_ops)]
    asg = np.array([[rng.randrange(S[i]) for i in range(f.num_ops)] for _ in range(6)], np.int32)
    rc, rv, rm = B.reference_price_assignments(f, t, asg)
    for j in range(len(asg)):
        c, v, m = ref_price(f, ref, asg[j])
        assert (c, v, m) == (rc[j], rv[j], rm[j])


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_price_assignments_configs(cfg):
    g, t = getattr(M, cfg)()
    check(g, t, 64, 3)


@pytest.mark.gpu
def test_price_assignments_gpt_chain():
    g, t = M.cfg3(2)
    check(g, t, 16, 4)


@pytest.mark.gpu
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
