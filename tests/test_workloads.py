"""The seeded synthetic inputs (workloads/) match the recipes of BASELINE.json's configs
(DESIGN.md §6): CPU only."""
import numpy as np

from workloads import (dodecahedron, face_cycles, paper_graph, random_3perm, random_3perm_batch,
                       random_fullerene, truncated_icosahedron)


def _cubic_simple(a):
    return (a == a.T).all() and (np.diag(a) == 0).all() and (a.sum(0) == 3).all() and set(np.unique(a)) <= {0, 1}


def test_dodecahedron_c20():
    a = dodecahedron()
    assert a.shape == (20, 20) and _cubic_simple(a)
    assert face_cycles(a, 5) == 12  # 12 pentagonal faces


def test_truncated_icosahedron_c60():
    a = truncated_icosahedron()
    assert a.shape == (60, 60) and _cubic_simple(a)
    assert face_cycles(a, 5) == 12 and face_cycles(a, 6) == 20
    b = paper_graph("C60")
    assert _cubic_simple(b) and face_cycles(b, 5) == 12 and face_cycles(b, 6) == 20


def test_config2_batch():
    m = random_3perm_batch(256, 24, seed=2024)
    assert m.shape == (256, 24, 24)
    nz = m != 0
    assert (nz.sum(1) == 3).all() and (nz.sum(2) == 3).all()
    assert set(np.unique(m[:128])) == {0, 1}
    w = m[128:][nz[128:]]
    assert w.min() >= 1 and w.max() <= 7 and len(np.unique(w)) == 7
    assert (random_3perm_batch(256, 24, seed=2024) == m).all()  # seeded


def test_random_3perm_disjoint():
    rng = np.random.default_rng(0)
    a = random_3perm(96, rng)
    assert ((a != 0).sum(0) == 3).all() and ((a != 0).sum(1) == 3).all() and set(np.unique(a)) == {0, 1}


def test_spiral_fullerenes_config4():
    for n in (70, 76):
        for iso in range(2):
            a, pos = random_fullerene(n, 2024, iso)
            assert a.shape == (n, n) and _cubic_simple(a)
            assert face_cycles(a, 5) == 12
            assert face_cycles(a, 6) == n // 2 - 10
