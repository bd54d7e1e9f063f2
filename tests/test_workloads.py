"""Generator sanity (host logic, CPU): sizes per SURVEY §8(d), determinism, Q-readings."""
import numpy as np
import pytest

from workloads import gen


@pytest.mark.parametrize("cfg,N,T,L", [(1, 25, 10, 3), (2, 3600, 60, 32), (3, 20000, 100, 256),
                                        (4, 40000, 200, 1024), (5, 5000, 100, 8192)])
def test_config_shapes_and_readings(cfg, N, T, L):
    p = gen(cfg)
    assert (p.N, p.T, p.L) == (N, T, L)
    loops = p.tail == p.head
    assert loops.sum() == N                                   # Q1: one self-loop per node
    assert np.all(np.isinf(p.cap[loops]))                     # Q4: loops uncapacitated
    assert np.all(np.isfinite(p.cap[~loops]))
    key = p.tail.astype(np.int64) * p.N + p.head
    assert np.unique(key).size == p.A                         # no duplicate arcs
    assert np.all(np.isfinite(p.cost)) and np.all(p.cost >= 0)
    if cfg == 1:
        assert p.A == 105 and p.prec == "fp64"
    if cfg == 2:
        assert p.A == 17760
        assert np.allclose(p.mu0.sum(1), 1.0) and np.allclose(p.muT.sum(1), 1.0)
    if p.is_point:
        assert np.all(p.src != p.dst)
    if cfg == 5:
        assert np.allclose(p.mass, 1.0 / L)


def test_deterministic():
    a, b = gen(3), gen(3)
    assert np.array_equal(a.tail, b.tail) and np.array_equal(a.cost, b.cost) and np.array_equal(a.src, b.src)


def test_lite_commodities_are_prefix():
    full, lite = gen(5), gen(5, L=64)
    assert np.array_equal(full.tail, lite.tail)
    # caps scale with the overriding L (Q18), OD list is a prefix
    assert np.array_equal(full.src[:64], lite.src) and np.array_equal(full.dst[:64], lite.dst)
