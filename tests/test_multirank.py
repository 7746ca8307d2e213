"""N>1 host logic on CPU (gloo, world_size 2): edge-range partitioning, and
a sharded build whose per-rank slices, gathered point-to-point onto rank 0,
reproduce the full build. The per-rank compute here is the oracle (this is
the CPU stand-in for the CUDA engine the GPU ranks call)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_04285_b200 import distributed as D, graph as G, models as M


def test_partition_edges_balanced_and_contiguous():
    counts = [196, 1806, 1806, 1806, 1806, 196, 196, 1806] * 20
    for world in (1, 2, 3, 4, 8):
        r = D.partition_edges(counts, world)
        assert r[0][0] == 0 and r[-1][1] == len(counts)
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        loads = [sum(counts[a:b]) for a, b in r]
        assert max(loads) - min(loads) <= 2 * max(counts)


def test_partition_scenarios_lpt():
    costs = [5, 1, 9, 3, 3, 7, 2]
    parts = D.partition_scenarios(costs, 3)
    assert sorted(i for p in parts for i in p) == list(range(len(costs)))
    loads = sorted(sum(costs[i] for i in p) for p in parts)
    assert loads[-1] - loads[0] <= max(costs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(flat, topo, rng):
    from oracle import bindings as B
    full = B.oracle_build(flat, topo, records=False)
    ix = dict(node_base=full.node_base, edge_base=full.edge_base, edge_from_op=full.edge_from_op,
              edge_to_op=full.edge_to_op)
    lo, hi = int(full.edge_base[rng[0]]), int(full.edge_base[rng[1]])
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a[lo:hi]))
    return ix, t(full.edge_cost_s), t(full.edge_volume_bytes), t(full.edge_memory_bytes)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, t = M.cfg2()
    f = G.flatten(g)
    ranges, out = D.sharded_build(dist, f, t, _oracle_compute, gather=True)
    if rank == 0:
        q.put((ranges, [x.numpy().copy() for x in out]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_build_gathers_full_tensors():
    from oracle import bindings as B
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ranges, (c, v, m) = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g, t = M.cfg2()
    full = B.oracle_build(G.flatten(g), t, records=False)
    assert ranges[0][0] == 0 and ranges[-1][1] == len(g.edges) and ranges[0][1] == ranges[1][0]
    assert np.array_equal(c.view(np.uint64), full.edge_cost_s.view(np.uint64))
    assert np.array_equal(v.view(np.uint64), full.edge_volume_bytes.view(np.uint64))
    assert np.array_equal(m.view(np.uint64), full.edge_memory_bytes.view(np.uint64))
