"""Pins of the BKW workload's host side (paper_1201_3986_b200.bkw) against the
closed form of PAPER.md:959-967: unit mass and energy 2 for all t, S(0) = 1/2,
positivity, and the analytic time derivative against a finite difference."""
import math

import numpy as np
import pytest

from paper_1201_3986_b200 import bkw


def _moments(t, N=256, T=12.0):
    v2 = bkw.grid_v2(N, T)
    h = 2 * T / N
    f = bkw.f_exact(t, v2)
    return f, h * h * f.sum(), h * h * (v2 * f).sum()


@pytest.mark.parametrize("t", [0.0, 0.5, 3.0, 40.0])
def test_bkw_mass_energy_positivity(t):
    f, m, e = _moments(t)
    assert abs(m - 1.0) < 1e-10          # ∫ f = 1
    assert abs(e - 2.0) < 1e-9           # ∫ |v|^2 f = 2 (temperature 1 in 2D)
    assert f.min() >= 0.0


def test_bkw_s_and_derivative():
    assert bkw.S(0.0) == 0.5 and abs(bkw.S(1e9) - 1.0) < 1e-12
    v2 = bkw.grid_v2(64, 8.0)
    for t in (0.0, 0.7, 5.0):
        eps = 1e-5
        fd = (bkw.f_exact(t + eps, v2) - bkw.f_exact(t - eps, v2)) / (2 * eps)
        np.testing.assert_allclose(bkw.dfdt_exact(t, v2), fd, rtol=0, atol=1e-9)
    # the datum at t = 0 is |v|^2 exp(-|v|^2) / pi
    np.testing.assert_allclose(bkw.f_exact(0.0, v2), v2 * np.exp(-v2) / math.pi, rtol=1e-14, atol=1e-300)


def test_e1_definition():
    a = np.array([1.0, -2.0, 3.0])
    assert bkw.e1(a, a) == 0.0
    assert abs(bkw.e1(a, a + [0.5, 0.0, -0.5]) - 1.0 / 6.0) < 1e-15
