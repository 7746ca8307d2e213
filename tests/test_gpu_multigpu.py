"""N-GPU edge sharding of one build: every rank builds its
contiguous edge range with the CUDA engine into device memory, NCCL
point-to-point sends gather the slices onto rank 0 over NVLink, and the
result is bit-identical to the oracle's full build. Needs >= 2 GPUs (run with
`gpurun --gpus 2`); skipped on a single-GPU box."""
import os
import socket

import numpy as np
import pytest
import torch

from paper_2301_04285_b200 import distributed as D, graph as G, models as M

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    g, t = getattr(M, cfg)()
    f = G.flatten(g)
    ranges, out = D.sharded_build(dist, f, t, D.engine_compute(rank), gather=True)
    torch.cuda.synchronize()
    if rank == 0:
        q.put((ranges, [x.cpu().numpy().copy() for x in out]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
def test_edge_sharded_build_nccl_gather(cfg):
    import torch.multiprocessing as mp

    from oracle import bindings as B
    world = torch.cuda.device_count()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    ranges, (c, v, m) = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g, t = getattr(M, cfg)()
    full = B.oracle_build(G.flatten(g), t, records=False)
    assert ranges[0][0] == 0 and ranges[-1][1] == len(g.edges)
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    assert np.array_equal(c.view(np.uint64), full.edge_cost_s.view(np.uint64))
    assert np.array_equal(v.view(np.uint64), full.edge_volume_bytes.view(np.uint64))
    assert np.array_equal(m.view(np.uint64), full.edge_memory_bytes.view(np.uint64))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_batches_on_a_second_device():
    """The batch entry points on device 1 from a process whose current device
    is 0: every buffer (pooled arenas, the batch pack, the worker threads'
    allocations) must land on the plans' device."""
    from oracle import bindings as B
    from paper_2301_04285_b200 import engine
    torch.cuda.set_device(0)
    scen = M.scenario_sweep(60)
    pairs = [(G.flatten(s.graph), s.topo) for s in scen]
    res = engine.build_sweep(pairs, device=1, host_threads=4)
    ds = engine.DeviceSweep(pairs[:30], device=1)
    ds.run()
    torch.cuda.synchronize(1)
    ds.check_errors()
    for i, (f, t) in enumerate(pairs):
        ref = B.oracle_build(f, t, records=False)
        for k in ("node_intra_cost_s", "edge_cost_s", "edge_volume_bytes", "edge_memory_bytes"):
            assert np.array_equal(getattr(res[i], k).view(np.uint64), getattr(ref, k).view(np.uint64)), (i, k)
            if i < 30:
                got = ds.result(i)[k].cpu().numpy()
                assert np.array_equal(got.view(np.uint64), getattr(ref, k).view(np.uint64)), (i, k)
