"""Synthetic operator graphs of the five benchmark configurations.

The single-layer builders restate the reference's models.hpp
(/root/reference/proj/include/topoplan/models.hpp:49-304) and are checked
against it by tests/test_models.py (through oracle/_ref). The reference
emits one transformer layer only; `build_gpt_chain` composes
L of them for cfg3/cfg4, and `scenario_sweep` draws cfg5's
1,000 scenarios with the survey's seeded draw order.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

from .graph import (AxisSlice, ClusterTopology, ComputationGraph, GraphEdge, OperatorAxis,
                    OperatorNode, TensorSpec)


@dataclass
class ModelConfig:  # models.hpp:39-45
    family: str = "mlp-chain"
    hidden: int = 1024
    layers: int = 2
    batch: int = 64
    seq: int = 512


def _axis(name, slices):
    return OperatorAxis(name, [AxisSlice(t, d) for t, d in slices])


def dense_op(id, kind, in_name, rows, in_, out, out_name, out_rows=-1, out_cols=-1):
    """models.hpp:66-85: activation (rows, in) x weight (in, out)."""
    if out_rows < 0:
        out_rows = rows
    if out_cols < 0:
        out_cols = out
    w = id + ".w"
    return OperatorNode(
        id=id, kind=kind,
        inputs=[TensorSpec(in_name, [rows, in_]), TensorSpec(w, [in_, out])],
        outputs=[TensorSpec(out_name, [out_rows, out_cols])],
        axes=[_axis("b", [(in_name, 0), (out_name, 0)]),
              _axis("in", [(in_name, 1), (w, 0)]),
              _axis("out", [(w, 1), (out_name, 1)])])


def pointwise_op(id, in_name, out_name, rows, cols):
    """models.hpp:88-102."""
    return OperatorNode(
        id=id, kind="elementwise",
        inputs=[TensorSpec(in_name, [rows, cols])],
        outputs=[TensorSpec(out_name, [rows, cols])],
        axes=[_axis("d0", [(in_name, 0), (out_name, 0)]),
              _axis("d1", [(in_name, 1), (out_name, 1)])])


def build_mlp_chain(cfg: ModelConfig) -> ComputationGraph:  # models.hpp:106-121
    g = ComputationGraph()
    for l in range(cfg.layers):
        in_name, out_name = f"act{l}", f"act{l + 1}"
        g.operators.append(dense_op(f"fc{l + 1}", "matmul", in_name, cfg.batch, cfg.hidden,
                                    cfg.hidden, out_name))
        if l > 0:
            g.edges.append(GraphEdge(f"fc{l}", f"fc{l + 1}", in_name))
    return g


def _transformer_ops(h: int, rows: int, p: str, x_name: str):
    """One pre-norm layer (models.hpp:125-197) with every id/tensor prefixed
    by `p` and the layer input named `x_name`."""
    n = lambda s: p + s
    ops = [pointwise_op(n("ln1"), x_name, n("ln1_out"), rows, h)]
    for proj in ("q", "k", "v"):
        ops.append(dense_op(n(f"{proj}_proj"), "matmul", n("ln1_out"), rows, h, h, n(f"{proj}_out")))
    ops.append(OperatorNode(
        id=n("attn"), kind="other",
        inputs=[TensorSpec(n("q_out"), [rows, h]), TensorSpec(n("k_out"), [rows, h]),
                TensorSpec(n("v_out"), [rows, h])],
        outputs=[TensorSpec(n("attn_out"), [rows, h])],
        axes=[_axis("b", [(n("q_out"), 0), (n("k_out"), 0), (n("v_out"), 0), (n("attn_out"), 0)]),
              _axis("heads", [(n("q_out"), 1), (n("k_out"), 1), (n("v_out"), 1), (n("attn_out"), 1)])]))
    ops.append(dense_op(n("out_proj"), "matmul", n("attn_out"), rows, h, h, n("proj_out")))
    ops.append(OperatorNode(
        id=n("add1"), kind="elementwise",
        inputs=[TensorSpec(n("proj_out"), [rows, h]), TensorSpec(n("ln1_out"), [rows, h])],
        outputs=[TensorSpec(n("add1_out"), [rows, h])],
        axes=[_axis("d0", [(n("proj_out"), 0), (n("ln1_out"), 0), (n("add1_out"), 0)]),
              _axis("d1", [(n("proj_out"), 1), (n("ln1_out"), 1), (n("add1_out"), 1)])]))
    ops.append(pointwise_op(n("ln2"), n("add1_out"), n("ln2_out"), rows, h))
    ops.append(dense_op(n("mlp_fc"), "matmul", n("ln2_out"), rows, h, 4 * h, n("fc_out")))
    ops.append(pointwise_op(n("gelu"), n("fc_out"), n("gelu_out"), rows, 4 * h))
    ops.append(dense_op(n("mlp_proj"), "matmul", n("gelu_out"), rows, 4 * h, h, n("mlp_out")))
    ops.append(OperatorNode(
        id=n("add2"), kind="elementwise",
        inputs=[TensorSpec(n("mlp_out"), [rows, h]), TensorSpec(n("add1_out"), [rows, h])],
        outputs=[TensorSpec(n("add2_out"), [rows, h])],
        axes=[_axis("d0", [(n("mlp_out"), 0), (n("add1_out"), 0), (n("add2_out"), 0)]),
              _axis("d1", [(n("mlp_out"), 1), (n("add1_out"), 1), (n("add2_out"), 1)])]))
    pairs = [("ln1", "q_proj", "ln1_out"), ("ln1", "k_proj", "ln1_out"),
             ("ln1", "v_proj", "ln1_out"), ("q_proj", "attn", "q_out"),
             ("k_proj", "attn", "k_out"), ("v_proj", "attn", "v_out"),
             ("attn", "out_proj", "attn_out"), ("out_proj", "add1", "proj_out"),
             ("ln1", "add1", "ln1_out"), ("add1", "ln2", "add1_out"),
             ("ln2", "mlp_fc", "ln2_out"), ("mlp_fc", "gelu", "fc_out"),
             ("gelu", "mlp_proj", "gelu_out"), ("mlp_proj", "add2", "mlp_out"),
             ("add1", "add2", "add1_out")]
    edges = [GraphEdge(n(a), n(b), n(t)) for a, b, t in pairs]
    return ops, edges


def build_transformer_layer(cfg: ModelConfig) -> ComputationGraph:  # models.hpp:125-197
    ops, edges = _transformer_ops(cfg.hidden, cfg.batch * cfg.seq, "", "x")
    return ComputationGraph(ops, edges)


def build_gpt_chain(layers: int, hidden: int, batch: int, seq: int) -> ComputationGraph:
    """`layers` transformer layers in a chain: layer l's ops/tensors are
    prefixed "L{l}."; layer l+1's ln1 consumes layer l's add2_out
    (SURVEY.md §8d cfg3/cfg4)."""
    g = ComputationGraph()
    rows = batch * seq
    x = "x"
    for l in range(layers):
        p = f"L{l}."
        ops, edges = _transformer_ops(hidden, rows, p, x)
        if l > 0:
            g.edges.append(GraphEdge(f"L{l - 1}.add2", p + "ln1", x))
        g.operators.extend(ops)
        g.edges.extend(edges)
        x = p + "add2_out"
    return g


def build_alexnet_like(cfg: ModelConfig) -> ComputationGraph:  # models.hpp:205-244
    b = cfg.batch
    layers = [("conv1", "conv", b * 55 * 55, 384, 64),
              ("conv2", "conv", b * 27 * 27, 64 * 25, 192),
              ("conv3", "conv", b * 13 * 13, 192 * 9, 384),
              ("conv4", "conv", b * 13 * 13, 384 * 9, 256),
              ("conv5", "conv", b * 13 * 13, 256 * 9, 256),
              ("fc6", "matmul", b, 256 * 36, 4096),
              ("fc7", "matmul", b, 4096, 4096),
              ("fc8", "matmul", b, 4096, 1024)]
    g = ComputationGraph()
    for i, (id, kind, rows, in_, out) in enumerate(layers):
        out_rows = out_cols = -1
        if i + 1 < len(layers):
            out_rows, out_cols = layers[i + 1][2], layers[i + 1][3]
        g.operators.append(dense_op(id, kind, f"act{i}", rows, in_, out, f"act{i + 1}",
                                    out_rows, out_cols))
        if i > 0:
            g.edges.append(GraphEdge(layers[i - 1][0], id, f"act{i}"))
    return g


def build_graph(cfg: ModelConfig) -> ComputationGraph:  # models.hpp:246-256
    if cfg.hidden < 1 or cfg.layers < 1 or cfg.batch < 1 or cfg.seq < 1:
        raise ValueError("model config sizes must be positive")
    return {"mlp-chain": build_mlp_chain, "transformer-layer": build_transformer_layer,
            "alexnet-like": build_alexnet_like}[cfg.family](cfg)


def parse_model_spec(spec: str) -> ModelConfig:  # models.hpp:260-304
    family, _, params = spec.partition(":")
    defaults = {"mlp-chain": dict(hidden=1024, layers=2, batch=256),
                "transformer-layer": dict(hidden=2304, batch=8, seq=512),
                "alexnet-like": dict(batch=64)}
    if family not in defaults:
        raise ValueError(f"unknown model family '{family}'")
    cfg = ModelConfig(family=family, **defaults[family])
    for kv in filter(None, params.split(",")):
        key, eq, val = kv.partition("=")
        if not eq:
            raise ValueError(f"bad model parameter '{kv}' (expected key=value)")
        if key not in ("hidden", "layers", "batch", "seq"):
            raise ValueError(f"unknown model parameter '{key}'")
        setattr(cfg, key, int(val))
    return cfg


def topology(nodes: int, local: int, intra_gbps: float = 60, inter_gbps: float = 6,
             mem_gb: float = 80) -> ClusterTopology:
    return ClusterTopology(nodes, local, intra_gbps * 1e9, inter_gbps * 1e9, mem_gb * 1e9)


def sample_graph() -> ComputationGraph:
    """data/sample_graph.json (fc1 -> relu -> fc2), cfg1's graph."""
    fc1 = dense_op("fc1", "matmul", "x0", 256, 1024, 4096, "x1")
    relu = pointwise_op("relu", "x1", "x2", 256, 4096)
    fc2 = dense_op("fc2", "matmul", "x2", 256, 4096, 1024, "x3")
    return ComputationGraph([fc1, relu, fc2],
                            [GraphEdge("fc1", "relu", "x1"), GraphEdge("relu", "fc2", "x2")])


# --------------------------------------------------------------------------
# the benchmark configurations
# --------------------------------------------------------------------------

def cfg1():
    return sample_graph(), ClusterTopology(2, 4, 60e9, 6e9, 32e9)


def cfg2():
    g = build_transformer_layer(ModelConfig("transformer-layer", hidden=4096, batch=8, seq=512))
    return g, topology(4, 8)


CFG3_RATIOS = (1, 2, 5, 10, 20, 50, 100)


def cfg3(nodes: int = 8, ratio: float = 10):
    return build_gpt_chain(24, 2048, 8, 512), ClusterTopology(nodes, 8, 60e9, 60e9 / ratio, 80e9)


def cfg4(ratio: float = 10):
    return build_gpt_chain(96, 12288, 8, 2048), ClusterTopology(16, 8, 60e9, 60e9 / ratio, 80e9)


class MT19937_64:
    """std::mt19937_64, for cfg5's seeded scenario draw."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) \
                & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def __call__(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


@dataclass
class Scenario:
    family: str
    params: dict
    graph: ComputationGraph
    topo: ClusterTopology


def scenario_sweep(count: int = 1000, seed: int = 0x230104285) -> List[Scenario]:
    """cfg5: `count` (model, mesh, bandwidth-ratio) scenarios with the draw
    order of SURVEY.md §8d."""
    rng = MT19937_64(seed)
    out = []
    for _ in range(count):
        fam = rng() % 4
        nodes = 1 << (rng() % 4)
        ratio = 10 ** ((rng() % 1001) / 500.0)
        if fam == 0:
            layers = 2 + rng() % 7
            hidden = 256 << (rng() % 5)
            params = dict(layers=layers, hidden=hidden, batch=256)
            g = build_mlp_chain(ModelConfig("mlp-chain", hidden=hidden, layers=layers, batch=256))
            name = "mlp-chain"
        elif fam == 1:
            hidden = 1024 << (rng() % 3)
            params = dict(hidden=hidden, batch=8, seq=512)
            g = build_transformer_layer(ModelConfig("transformer-layer", hidden=hidden, batch=8, seq=512))
            name = "transformer-layer"
        elif fam == 2:
            params = dict(batch=64)
            g = build_alexnet_like(ModelConfig("alexnet-like", batch=64))
            name = "alexnet-like"
        else:
            layers = 2 + rng() % 3
            params = dict(layers=layers, hidden=2048, batch=8, seq=512)
            g = build_gpt_chain(layers, 2048, 8, 512)
            name = "gpt-chain"
        params["ratio"] = ratio
        topo = ClusterTopology(nodes, 8, 60e9, 60e9 / ratio, 80e9)
        out.append(Scenario(name, params, g, topo))
    return out


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}
