"""§8(f)3: the reference's wire formats written straight from the cost
tensors -- export_lp (solver.hpp:578-600, "%.17g") and aux_graph_to_json
(io.hpp:208-239) -- byte-identical to the reference's own output.

CPU: oracle/_ref/export_parity pins the writers of
include/taps_b200/export_b200.hpp (+ lp_export.hpp) to the reference on
reference-built graphs. GPU: tp_plan_export_lp writes the LP of an
engine-built plan from its host SoA tensors; the C++ adapter's JSON / LP of
GPU-built graphs are checked in oracle/adapter_parity.cpp."""
import os
import subprocess

import pytest

from oracle import bindings as B
from paper_2301_04285_b200 import engine, fuzz, graph as G, models as M

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "oracle", "_ref", "export_parity")


@pytest.mark.skipif(not os.path.exists(BIN), reason="export_parity not built (needs /root/reference at build time)")
def test_writers_match_reference_on_cpu():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "[EXPORT] ALL PASS" in r.stdout


def _check_lp(g, t, tmp_path):
    f = G.flatten(g)
    plan = engine.Plan(f, t, device=0)
    ct = plan.execute_host()
    for vol in (False, True):
        path = str(tmp_path / f"b200_{int(vol)}.lp")
        n = plan.export_lp(ct, path, mode="volume" if vol else "topology")
        got = open(path, "rb").read()
        assert len(got) == n
        ref = B.reference_export_lp(f, t, mode_volume=vol)
        assert got == ref, f"LP text differs (volume={vol}) at byte {next(i for i in range(min(len(got), len(ref))) if got[i] != ref[i]) if got[:len(ref)] != ref[:len(got)] else min(len(got), len(ref))}"


@pytest.mark.gpu
@pytest.mark.skipif(not B.have_reference(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_export_lp_from_device_tensors(cfg, tmp_path):
    g, t = M.cfg3(2) if cfg == "cfg3" else getattr(M, cfg)()
    _check_lp(g, t, tmp_path)


@pytest.mark.gpu
@pytest.mark.skipif(not B.have_reference(), reason="oracle/_ref not built")
def test_export_lp_random_graphs(tmp_path):
    import random
    rng = random.Random(17)
    done = 0
    for i in range(60):
        g, t = fuzz.random_planning_instance(rng)
        if B.oracle_build(G.flatten(g), t).status != 0:
            continue
        _check_lp(g, t, tmp_path)
        done += 1
    assert done >= 10
