"""The seeded generators: determinism and the brute-force counts the configs are quoted on."""
import numpy as np

import synth
from helpers import golden


def test_determinism():
    a = synth.large_D(1000)
    b = synth.large_D(1000)
    assert np.array_equal(a, b)
    assert not np.array_equal(synth.rng("a").random(4), synth.rng("b").random(4))


def test_config_space_counts():
    """SPEC.md:395 (51); 3-D pow2 with bz <= 64: 266, 231 after the warp rule; F_large: 1,024
    with 464 statically feasible (brute force)."""
    assert len(synth.F_pow2_2d()) == golden("spec_worked.json")["config_space"][0]["count"] == 51
    F3 = synth.F_pow2_3d()
    assert len(F3) == 266 and int(np.sum(F3.prod(1) % 32 == 0)) == 231
    FL = synth.F_large()
    T = FL.prod(1)
    assert len(FL) == 1024 and int(np.sum((T % 32 == 0) & (T <= 1024))) == 464
    # filter by bx*by <= N*N at N = 8 keeps products {32, 64}
    F2 = synth.F_pow2_2d()
    assert sorted(set(F2.prod(1)[F2.prod(1) <= 64].tolist())) == [32, 64]


def test_bases():
    b = synth.basis_total_degree(1, 1)
    assert b.tolist() == [[0], [1]]
    assert len(synth.basis_total_degree(4, 4)) == 70 and len(synth.basis_total_degree(4, 3)) == 35
    assert synth.basis_box([1, 1]).tolist() == [[0, 0], [0, 1], [1, 0], [1, 1]]
    b = synth.basis_total_degree(3, 2)
    assert b[0].tolist() == [0, 0, 0] and np.all(np.diff(b.sum(1)) >= 0)


def test_classf_bounds():
    g = synth.rng("t", "classf")
    basis = synth.basis_total_degree(4, 4)
    c = synth.classf_coefficients(g, basis, 1.0)
    a, b = c[:70], c[70:]
    assert b[0] == 1.0 and abs(np.abs(b[1:]).sum() - 0.5) < 1e-15
    assert a[0] >= 1.0 + np.abs(a[1:]).sum() - 1e-12
    assert np.all(c != 0)


def test_sizes():
    assert synth.tiny_sizes().ravel().tolist()[:4] == [8, 12, 16, 24] and len(synth.tiny_sizes()) == 16
    D = synth.large_D(10000)
    assert D.min() >= 8 and D.max() <= 16384
    X = synth.box_random_design(synth.rng("t"), *synth.LARGE_BOX, 100)
    assert X[0].tolist() == synth.LARGE_BOX[0] and X[1].tolist() == synth.LARGE_BOX[1]
