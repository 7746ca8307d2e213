"""The C-ABI library without a GPU: it loads, exports every function the
header declares, and fails loudly (TP_ERR_CUDA) instead of falling back to
a CPU path."""
import ctypes as C
import os
import re

import pytest
import torch

from paper_2301_04285_b200 import abi, engine, graph as G, models as M

HEADER = os.path.join(abi.REPO_DIR, "include", "taps_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:tp_status|void|int32_t|int64_t|const char\*)\s+(tp_\w+)\(", text, re.M)))


def test_header_declarations_are_exported(engine):
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(engine, n), n
    assert set(abi.EXPORTED_SYMBOLS) <= set(names)


def test_abi_version(engine):
    assert engine.tp_abi_version() == abi.TP_ABI_VERSION == 2


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly():
    g, t = M.cfg1()
    with pytest.raises(RuntimeError, match="no CUDA device"):
        engine.build_cost_tensors(g, t)
    with pytest.raises(RuntimeError):
        engine.enumerate_strategies(3, 4)


def test_engine_missing_is_an_error(monkeypatch, tmp_path):
    monkeypatch.setattr(abi, "ENGINE_SO", str(tmp_path / "nope.so"))
    monkeypatch.setattr(abi, "_engine", None)
    with pytest.raises(abi.EngineMissing):
        abi.load_engine()


def test_strategy_count_query_needs_no_gpu(engine):
    n = C.c_int64()
    assert engine.tp_enumerate_strategies(3, 128, C.byref(n), None, None, None, None) == 0
    assert n.value == 129
    assert engine.tp_enumerate_strategies(3, 6, C.byref(n), None, None, None, None) == abi.TP_ERR_TOPOPLAN


STRUCTS = ("tp_graph_desc", "tp_topology_desc", "tp_aux_index", "tp_cost_tensors", "tp_build_opts",
           "tp_plan_sizes_t", "tp_redist_query", "tp_redist_result")


def test_ctypes_structs_match_the_header(tmp_path):
    """Every ctypes mirror in abi.py has the C header's size and field offsets
    (a field appended to the header but not to abi.py would shift everything
    the Python side passes across the ABI)."""
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {"]
    for s in STRUCTS:
        lines.append(f'  printf("{s} sizeof %zu\\n", sizeof({s}));')
        for f, _ in getattr(abi, s)._fields_:
            lines.append(f'  printf("{s} {f} %zu\\n", offsetof({s}, {f}));')
    lines += ["  return 0;", "}"]
    src, exe = tmp_path / "probe.c", tmp_path / "probe"
    src.write_text("\n".join(lines) + "\n")
    import subprocess
    subprocess.run(["gcc", "-std=c99", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for s in STRUCTS:
        cls = getattr(abi, s)
        assert got[(s, "sizeof")] == C.sizeof(cls), s
        for f, _ in cls._fields_:
            assert got[(s, f)] == getattr(cls, f).offset, (s, f)
