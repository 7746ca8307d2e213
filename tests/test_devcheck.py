"""Kernel-logic check without a GPU: the engine's per-pair algorithms
(tp_core.cuh array form, tp_fast.cuh register form — the code the kernels
run) compiled for the host (tests/devcheck/core_host.cpp) against the
oracle. The product library has no CPU path; this build exists only here."""
import ctypes as C
import random

import numpy as np
import pytest

from oracle import bindings as B
from paper_2301_04285_b200 import abi, fuzz
from paper_2301_04285_b200.build import build_devcheck


@pytest.fixture(scope="module")
def core():
    lib = C.CDLL(build_devcheck())
    for fn in ("core_redistribute", "core_redistribute_fast"):
        getattr(lib, fn).argtypes = [C.POINTER(abi.tp_redist_query), C.POINTER(abi.tp_redist_result)]
        getattr(lib, fn).restype = C.c_int
    lib.core_unrank.argtypes = [C.c_int, C.c_int, C.c_longlong] + [C.POINTER(C.c_int)] * 4
    return lib


def run(lib, fn, q):
    r = abi.tp_redist_result()
    getattr(lib, fn)(C.byref(q), C.byref(r))
    return r


def same(a, b):
    return (a.plan() == b.plan() and a.volume_bytes == b.volume_bytes and a.seconds == b.seconds
            and list(a.op_seconds[: a.num_ops]) == list(b.op_seconds[: b.num_ops]))


def test_unranking_matches_enumeration(core):
    for p in range(1, 5):
        for N in (1, 2, 4, 8, 16, 32, 64, 128):
            deg, dm, md, dep = B.enumerate_with(B.oracle().oracle_enumerate, p, N)
            D, M_, X, d = (C.c_int * 8)(), (C.c_int * 8)(), (C.c_int * 8)(), C.c_int()
            for s in range(len(deg)):
                core.core_unrank(p, N.bit_length() - 1, s, D, M_, X, C.byref(d))
                assert [1 << D[a] for a in range(p)] == list(deg[s])
                assert [M_[a] for a in range(p)] == list(dm[s])


def cases(seed, n):
    rng = random.Random(seed)
    for i in range(n):
        total = 1 << rng.randrange(0, 8)

        def mat():
            d = fuzz.random_matrix_with_total(rng, total)
            if rng.randrange(3) == 0 and total > 1:
                d = [total]
            if rng.randrange(4) == 0:
                for _ in range(rng.randrange(1, 3)):
                    d.insert(rng.randrange(len(d) + 1), 1)
            return d
        d1, d2 = mat(), mat()
        rank = rng.randint(1, 4)
        shape = [rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 5, 10, 20, 7, 128, 256, 384])
                 for _ in range(rank)]

        def rm(dims):
            m = [-1] * rank
            for a in range(rank):
                if dims and rng.randrange(3):
                    m[a] = rng.randrange(len(dims))  # repeated device dims allowed
            return m
        yield B.make_query(shape, d1, rm(d1), d2, rm(d2), local=rng.choice([1, 2, 4, 8, 16, 32, 3]),
                           inter=rng.choice([6e9, 60e9, 1.5e9]))


@pytest.mark.parametrize("fn", ["core_redistribute", "core_redistribute_fast"])
def test_pair_algorithms_match_oracle(core, fn):
    ok = err = 0
    for qq in cases(11, 6000):
        a, b = B.oracle_redistribute(qq), run(core, fn, qq)
        assert a.status == b.status
        if a.status == 0:
            assert same(a, b)
            ok += 1
        else:
            err += 1
    assert ok > 2000 and err > 500


@pytest.mark.parametrize("fn", ["core_redistribute", "core_redistribute_fast"])
def test_pair_algorithms_on_reference_cases(core, fn):
    rng = random.Random(5)
    for i in range(4000):
        dims, shape, fm, tm = fuzz.random_redist_case(rng)
        if i % 2:
            d2 = fuzz.random_matrix_with_total(rng, int(np.prod(dims)))
            tm = fuzz.random_map_for(rng, shape, d2)
        else:
            d2 = dims
        qq = B.make_query(shape, dims, fm, d2, tm, local=rng.choice([1, 2, 4, 8]))
        a, b = B.oracle_redistribute(qq), run(core, fn, qq)
        assert a.status == b.status and (a.status or same(a, b))
