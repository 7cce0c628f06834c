"""Re-expresses proj/tests/test_contour.cpp and acceptance C1
(proj/tests/acceptance.cpp:65-94) against both the CPU oracle (pin) and the B200 path (F = b200, -m gpu)."""
import math

import numpy as np
import pytest

import oracle as O


def test_gauss_legendre_analytic_rules(F):
    x, w = F.gauss_legendre(1)
    assert abs(x[0]) <= 1e-15 and abs(w[0] - 2.0) <= 1e-15 * 2
    x, w = F.gauss_legendre(2)
    assert x[0] == pytest.approx(-1 / math.sqrt(3), rel=1e-14)
    assert x[1] == pytest.approx(1 / math.sqrt(3), rel=1e-14)
    assert w == pytest.approx([1.0, 1.0], rel=1e-14)
    x, w = F.gauss_legendre(3)
    assert x[0] == pytest.approx(-math.sqrt(0.6), rel=1e-14)
    assert x[1] == 0.0
    assert x[2] == pytest.approx(math.sqrt(0.6), rel=1e-14)
    assert w == pytest.approx([5 / 9, 8 / 9, 5 / 9], rel=1e-14)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 16, 24, 33, 48, 64])
def test_gauss_legendre_sum_and_symmetry(F, n):
    x, w = F.gauss_legendre(n)
    assert abs(w.sum() - 2.0) <= 1e-14
    assert np.all(np.diff(x) > 0)
    np.testing.assert_allclose(x, -x[::-1], rtol=1e-14, atol=0)
    np.testing.assert_allclose(w, w[::-1], rtol=1e-14, atol=0)


def test_gauss_legendre_rejects_out_of_range(F):
    with pytest.raises(F.InvalidArgument):
        F.gauss_legendre(0)
    with pytest.raises(F.InvalidArgument):
        F.gauss_legendre(65)


def test_single_node_rule(F):
    r = F.build_contour_rule(O.SearchInterval(-1, 1), 1)
    assert r.num_points() == 1
    assert abs(r.nodes[0] - 1j) <= 1e-15
    assert abs(r.weights[0] - 1j) <= 1e-15


def test_mapping_on_0_4(F):
    r = F.build_contour_rule(O.SearchInterval(0, 4), 2)
    for z in r.nodes:
        assert abs(abs(z - 2.0) - 2.0) <= 1e-14 * 2.0
        assert z.imag > 0
    t0 = np.angle(r.nodes[0] - 2.0)
    t1 = np.angle(r.nodes[1] - 2.0)
    assert t0 == pytest.approx(0.5 * math.pi * (1 - 1 / math.sqrt(3)), rel=1e-14)
    assert t1 == pytest.approx(0.5 * math.pi * (1 + 1 / math.sqrt(3)), rel=1e-14)


@pytest.mark.parametrize("nc", [1, 3, 8, 16])
def test_rule_invariants(F, nc):
    I = O.SearchInterval(-2.5, 0.75)
    r = F.build_contour_rule(I, nc)
    assert np.all(r.nodes.imag > 0)
    assert np.all(np.abs(np.abs(r.nodes - I.center()) - I.radius()) <= 1e-14 * I.radius())
    assert abs(F.filter_value(r, I.center()) - 1.0) <= 1e-14
    I2 = O.SearchInterval(-2.0, 1.5)
    r2 = F.build_contour_rule(I2, nc)
    assert abs(F.filter_value(r2, I2.center()) - 1.0) <= 1e-14
    for d in (0.3, 0.9, 2.1, 7.0):
        assert abs(F.filter_value(r2, I2.center() + d) - F.filter_value(r2, I2.center() - d)) <= 1e-14
    assert abs(F.filter_value(r2, I2.center() + 1e3 * I2.radius())) <= 1e-4


def test_filter_symmetry_endpoint_decay_plateau(F):
    r = F.build_contour_rule(O.SearchInterval(-1, 1), 8)
    for d in (0.1, 0.5, 0.93, 1.7, 12.0):
        assert abs(F.filter_value(r, d) - F.filter_value(r, -d)) <= 1e-14
    assert abs(F.filter_value(r, 1.0) - 0.5) <= 0.05
    assert O.exact_circle_filter(O.SearchInterval(-1, 1), 0.999999) == pytest.approx(1.0, rel=1e-4)
    assert abs(F.filter_value(r, 1000.0)) <= 1e-4
    r3 = F.build_contour_rule(O.SearchInterval(2, 6), 3)
    assert abs(F.filter_value(r3, 4.0 + 2000.0)) <= 1e-4
    for i in range(100):
        lam = -0.5 + i / 99.0
        assert abs(F.filter_value(r, lam) - 1.0) <= 1e-3


def test_nc16_matches_adaptive_integration(F):
    I = O.SearchInterval(-1, 1)
    r = F.build_contour_rule(I, 16)
    for lam in (0.0, 0.2, -0.35, 0.49, 1.5, -1.8, 2.5, 4.0, -7.0, 0.25, -0.4, -0.49, -1.6, 2.0, 3.5,
                -5.0, 9.0):
        assert abs(F.filter_value(r, lam) - O.exact_circle_filter(I, lam)) <= 1e-6


def test_predicted_rate(F):
    r = F.build_contour_rule(O.SearchInterval(-1, 1), 8)
    assert O.predicted_rate(r, [-0.5, 0.0, 0.5, 5.0, 9.0, 14.0], 3) < 0.01
    assert O.predicted_rate(r, [-0.5, 0.0, 0.5, 1.001, 1.002, 1.003], 4) > 0.9
    spec = [-0.7, 0.1, 0.6, 2.4]
    expected = F.filter_value(r, 2.4) / F.filter_value(r, -0.7)
    assert O.predicted_rate(r, spec, 3) == pytest.approx(expected, rel=1e-14)
    with pytest.raises(O.InvalidArgument):
        O.predicted_rate(r, spec, 4)
    with pytest.raises(O.InvalidArgument):
        O.predicted_rate(r, spec, 0)


def test_external_nodes(F):
    I = O.SearchInterval(-1, 1)
    base = F.build_contour_rule(I, 4)
    wrapped = F.contour_rule_from_nodes(I, base.nodes, base.weights)
    assert F.filter_value(wrapped, 0.3) == F.filter_value(base, 0.3)
    bad = base.nodes.copy()
    bad[0] = np.conj(bad[0])
    with pytest.raises(F.InvalidArgument):
        F.contour_rule_from_nodes(I, bad, base.weights)


def test_interval(F):
    with pytest.raises(F.InvalidArgument):
        F.SearchInterval(1.0, 1.0)
    with pytest.raises(F.InvalidArgument):
        F.SearchInterval(2.0, -1.0)
    I = F.SearchInterval(-1, 1)
    assert I.contains(0.0) and not I.contains(1.0) and not I.contains(-1.0)
