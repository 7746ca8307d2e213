"""The single-process multi-GPU build (tp_build_cost_tensors_multi /
tp_plan_execute_host_multi): edge ranges balanced by aux
edges, each device writing its slice straight into the caller's host arrays,
bit-identical to the one-device build and to the oracle. One device runs the
multi path's code on a 1-GPU box; the 2- and 4-device cases need the GPUs
(gpurun --gpus 2/4)."""
import numpy as np
import pytest

from golden_util import bits
from oracle import bindings as B
from paper_2301_04285_b200 import abi, engine, graph as G, models as M

pytestmark = pytest.mark.gpu

FIELDS = ("node_intra_cost_s", "node_intra_volume_bytes", "node_memory_bytes", "edge_cost_s",
          "edge_volume_bytes", "edge_memory_bytes", "row_min_cost_s", "row_min_volume_bytes",
          "edge_pair_min_cost_s", "edge_pair_min_volume_bytes")


def ndev():
    import torch
    return torch.cuda.device_count()


def check(got, ref, tag):
    for k in FIELDS:
        a, b = getattr(got, k), getattr(ref, k)
        assert a.shape == b.shape, (tag, k)
        assert np.array_equal(bits(a), bits(b)), f"{tag}: {k} differs"
    ne = len(ref.edge_cost_s)
    a, b = got.records[: ne * 40].reshape(-1, 40).copy(), ref.records.reshape(-1, 40).copy()
    a[:, 12:16] = 0
    b[:, 12:16] = 0
    assert np.array_equal(a, b), f"{tag}: records differ"


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_multi_matches_oracle(cfg, n):
    if ndev() < n:
        pytest.skip(f"needs {n} GPUs")
    g, t = M.cfg3(4) if cfg == "cfg3" else getattr(M, cfg)()
    f = G.flatten(g)
    got = engine.build_cost_tensors_multi(f, t, list(range(n)), records=True, row_min=True, pinned=True)
    check(got, B.oracle_build(f, t), f"{cfg} on {n}")


@pytest.mark.parametrize("n", [2, 4])
def test_multi_cfg4(n):
    if ndev() < n:
        pytest.skip(f"needs {n} GPUs")
    g, t = M.cfg4()
    f = G.flatten(g)
    ref = B.oracle_build(f, t, records=False)
    plan = engine.Plan(f, t, device=0)
    got = plan.execute_host_multi(list(range(n)), pinned=True)
    for k in FIELDS[:6]:
        assert np.array_equal(bits(getattr(got, k)), bits(getattr(ref, k))), k
    # re-executed (shards keep their arenas), then re-priced: still the oracle's
    plan.set_bandwidth(60e9, 60e9 / 50)
    got = plan.execute_host_multi(list(range(n)), pinned=True)
    ref = B.oracle_build(f, M.ClusterTopology(16, 8, 60e9, 60e9 / 50, 80e9), records=False)
    for k in FIELDS[:6]:
        assert np.array_equal(bits(getattr(got, k)), bits(getattr(ref, k))), k


def test_multi_errors_and_arguments():
    g = G.ComputationGraph([M.dense_op("fc", "matmul", "x", 6, 6, 6, "y")], [])
    t = G.ClusterTopology(1, 4, 60e9, 60e9, 32e9)
    with pytest.raises(abi.TopoplanError):
        engine.build_cost_tensors_multi(G.flatten(g), t, [0])
    g1, t1 = M.cfg1()
    with pytest.raises(ValueError):
        engine.build_cost_tensors_multi(G.flatten(g1), t1, [0, 0])
    with pytest.raises(ValueError):
        engine.build_cost_tensors_multi(G.flatten(g1), t1, [ndev()])
