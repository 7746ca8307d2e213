"""Multi-GPU sharding of the cost-tensor build.

One process per GPU. Two ways to split the work, neither with a collective on
the data path:
  * edge sharding of ONE build: contiguous ranges of graph edges balanced by
    their aux-edge counts sum(|Su| x |Sw|); each rank writes its contiguous
    slice [edge_base[e0], edge_base[e1]) of the global aux-edge arrays;
  * scenario sharding of a sweep (cfg5): whole (model, mesh, bandwidth)
    scenarios assigned longest-processing-time first.
The only communication is the optional gather of per-shard cost tensors onto
rank 0 (point-to-point sends, NCCL over NVLink on GPUs; gloo in the CPU
tests), used when the caller wants the full tensors on one device.
"""
from __future__ import annotations

import heapq
import math
from typing import Callable, List, Sequence, Tuple


def edge_pair_counts(node_base, edge_from_op, edge_to_op) -> List[int]:
    """|Su| * |Sw| of every graph edge (aux_graph.hpp:280-295)."""
    out = []
    for u, w in zip(edge_from_op, edge_to_op):
        su = int(node_base[u + 1] - node_base[u])
        sw = int(node_base[w + 1] - node_base[w])
        out.append(su * sw)
    return out


def partition_edges(pair_counts: Sequence[int], world: int) -> List[Tuple[int, int]]:
    """Contiguous edge ranges [e0, e1), one per rank, each as close as
    possible to 1/world of the aux edges (greedy split at the prefix-sum
    quantiles). Ranks may get empty ranges when edges < world."""
    n = len(pair_counts)
    total = sum(pair_counts)
    bounds = [0]
    acc = 0
    e = 0
    for r in range(1, world):
        target = total * r / world
        while e < n and acc + pair_counts[e] / 2 <= target:
            acc += pair_counts[e]
            e += 1
        bounds.append(max(e, bounds[-1]))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def strategy_count(p: int, total_devices: int) -> int:
    """layout.hpp:222-244 closed form: sum_i i! C(p,i) C(n-1,i-1)."""
    n = total_devices.bit_length() - 1
    if n == 0:
        return 1
    return sum(math.factorial(i) * math.comb(p, i) * math.comb(n - 1, i - 1) for i in range(1, min(p, n) + 1))


def estimated_aux_edges(graph, topo) -> int:
    """|E_A| of a scenario (sum over edges of S(from) * S(to)), the LPT weight
    of a sweep scenario; graph is a ComputationGraph."""
    N = topo.total_devices()
    S = [strategy_count(op.axis_count(), N) for op in graph.operators]
    return sum(S[graph.find_op(e.from_)] * S[graph.find_op(e.to)] for e in graph.edges)


def estimated_build_cost(graph, topo) -> float:
    """LPT weight of a sweep scenario on the device: its aux edges (the
    fan-out, ~12 ns each in a batch) plus its class-table entries (priced from
    op lists, ~70 ns each, fused_batch_kernel<5, 1> / <5, 2> measured on cfg5).
    Entries are estimated as S(from) * S(to) per distinct edge class (shape,
    bytes, slicing of both sides, axis counts -- aux_graph.hpp:257-271's memo
    key); the engine's layout dedup only makes them fewer."""
    N = topo.total_devices()
    S = [strategy_count(op.axis_count(), N) for op in graph.operators]
    aux = 0
    classes = set()
    pairs = 0
    for e in graph.edges:
        u, w = graph.find_op(e.from_), graph.find_op(e.to)
        aux += S[u] * S[w]
        ou, ow = graph.operators[u], graph.operators[w]
        spec = [t for t in list(ou.inputs) + list(ou.outputs) if t.name == e.tensor]
        if not spec:
            continue
        t = spec[-1]

        def slicing(op):
            m = [-1] * len(t.shape)
            for a, ax in enumerate(op.axes):
                for sl in ax.slices:
                    if sl.tensor == e.tensor and 0 <= sl.dim < len(m):
                        m[sl.dim] = a
            return tuple(m)
        key = (len(ou.axes), len(ow.axes), tuple(t.shape), t.element_size, slicing(ou), slicing(ow))
        if key not in classes:
            classes.add(key)
            pairs += S[u] * S[w]
    return float(aux) + 6.0 * pairs


def partition_scenarios(costs: Sequence[float], world: int) -> List[List[int]]:
    """Longest-processing-time assignment of scenarios to ranks; each rank's
    list keeps the scenarios' original order."""
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    assign: List[List[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda i: -costs[i]):
        load, r = heapq.heappop(heap)
        assign[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(a) for a in assign]


def gather_to_rank0(dist, local, ranges, edge_base, total, device=None, make_buffer=None):
    """Gather each rank's contiguous slice of a 1-D cost tensor onto rank 0.

    local: this rank's slice (a torch tensor); ranges: the edge ranges of all
    ranks; edge_base: aux-edge offsets. Rank 0 returns the full tensor, the
    others None. Point-to-point only (batch_isend_irecv)."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    if rank == 0:
        full = make_buffer(total) if make_buffer else torch.empty(total, dtype=local.dtype, device=local.device)
        e0, e1 = ranges[0]
        full[int(edge_base[e0]):int(edge_base[e1])] = local
        ops = []
        for r in range(1, world):
            a, b = ranges[r]
            lo, hi = int(edge_base[a]), int(edge_base[b])
            if hi > lo:
                ops.append(dist.P2POp(dist.irecv, full[lo:hi], r))
        for req in dist.batch_isend_irecv(ops) if ops else []:
            req.wait()
        return full
    a, b = ranges[rank]
    if int(edge_base[b]) > int(edge_base[a]):
        for req in dist.batch_isend_irecv([dist.P2POp(dist.isend, local.contiguous(), 0)]):
            req.wait()
    return None


def sharded_build(dist, flat, topo, compute: Callable, gather: bool = True):
    """Edge-sharded build of one graph. `compute(flat, topo, (e0, e1))` returns
    (index dict, edge_cost_s, edge_volume_bytes, edge_memory_bytes) of the
    rank's range as tensors — the CUDA engine on GPUs. Returns rank 0's
    gathered (cost, volume, memory) when gather=True, else the local slice."""
    rank, world = dist.get_rank(), dist.get_world_size()
    index, *_ = compute(flat, topo, (0, 0))
    counts = edge_pair_counts(index["node_base"], index["edge_from_op"], index["edge_to_op"])
    ranges = partition_edges(counts, world)
    index, c, v, m = compute(flat, topo, ranges[rank])
    if not gather:
        return ranges, (c, v, m)
    eb = index["edge_base"]
    total = int(eb[len(counts)])
    return ranges, tuple(gather_to_rank0(dist, x, ranges, eb, total) for x in (c, v, m))


def engine_compute(device: int):
    """The `compute` of sharded_build on a GPU rank: the CUDA engine builds the
    rank's edge range straight into device tensors (tp_plan_execute with
    tp_build_opts.edge_begin/end), ready for the NCCL gather."""
    import torch

    from . import engine as E

    import numpy as np

    cache = {}

    def content_key(flat, topo):
        # by content, not identity: a topology mutated in place (another
        # bandwidth) or a new FlatGraph at a recycled id() must not reuse a plan
        if not hasattr(flat, "desc"):
            from . import graph as G
            flat = G.flatten(flat)
        arrays = tuple(v.tobytes() for k, v in sorted(vars(flat).items()) if isinstance(v, np.ndarray))
        return (arrays, flat.num_ops, flat.num_edges, topo.node_count, topo.local_device_num,
                topo.intra_bandwidth, topo.inter_bandwidth, topo.device_memory), flat

    def compute(flat, topo, rng):
        key, flat = content_key(flat, topo)
        if key not in cache:
            cache.clear()
            cache[key] = E.Plan(flat, topo, device=device)
        plan = cache[key]
        ix = plan.index()
        e0, e1 = rng
        eb = ix["edge_base"]
        n = int(eb[e1] - eb[e0])
        dev = torch.device("cuda", device)
        outs = {k: torch.empty(max(n, 1), dtype=torch.float64, device=dev)
                for k in ("edge_cost_s", "edge_volume_bytes", "edge_memory_bytes")}
        stream = torch.cuda.current_stream(dev)
        if n > 0:
            plan.execute(E.device_cost_struct(outs), edge_range=(e0, e1), skip_nodes=True,
                         stream=stream.cuda_stream)
            plan.check_errors()
        return ix, outs["edge_cost_s"][:n], outs["edge_volume_bytes"][:n], outs["edge_memory_bytes"][:n]

    return compute
