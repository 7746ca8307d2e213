"""The C++ drop-in (include/taps_b200/aux_graph_b200.hpp) against the
reference, field by field, plus the reference's own ILP solver on both
(oracle/_ref/adapter_parity, built from /root/reference by oracle/Makefile)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "adapter_parity")


@pytest.mark.skipif(not os.path.exists(BIN), reason="adapter_parity not built (needs /root/reference at build time)")
def test_cpp_adapter_matches_reference_and_ilp():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "[PARITY] ALL PASS" in r.stdout
