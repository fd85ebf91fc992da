"""CPU pins of the oracle's Rician fidelity (PAPER App. D.3.3).
The Bessel ratio B = I1/I0 is pinned against its defining power series (written out here,
independent of the library routine the oracle calls) and the large-t asymptotic expansion; the
gradient against central finite differences of f; the special cases against the definitions."""
import math

import numpy as np
import pytest

from oracle import operators as ops
from oracle import solver as osolver
from paper_2605_19705_b200 import configs, synth


def _series_ratio(t, terms=80):
    """I0(t) = sum (t/2)^{2k} / (k!)^2, I1(t) = sum (t/2)^{2k+1} / (k! (k+1)!)."""
    i0 = i1 = 0.0
    for k in range(terms):
        a = (t / 2.0) ** (2 * k) / math.factorial(k) ** 2
        i0 += a
        i1 += a * (t / 2.0) / (k + 1)
    return i1 / i0


def test_bessel_ratio_power_series():
    ts = np.concatenate([[0.0, 1e-6, 0.1, 1.0], np.linspace(0.5, 15.0, 30)])
    for t in ts:
        want = _series_ratio(float(t))
        assert abs(ops.bessel_ratio(t) - want) <= 1e-10 * max(want, 1e-300)
    assert ops.bessel_ratio(0.0) == 0.0
    assert abs(ops.bessel_ratio(1.0) - 0.446390) < 5e-6            # SPEC worked value


def test_bessel_ratio_asymptotic_and_monotone():
    for t in (500.0, 700.0, 5000.0):                              # SPEC: B(500) within 1e-8
        assert abs(ops.bessel_ratio(t) - (1.0 - 1.0 / (2 * t) - 1.0 / (8 * t * t))) <= 1e-8
    g = np.linspace(0.0, 700.0, 100001)
    b = ops.bessel_ratio(g)
    assert np.all(np.isfinite(b)) and np.all(np.diff(b) >= 0) and np.all(b < 1.0)


def test_rician_gradient_finite_differences():
    rng = np.random.default_rng(3)
    sigma = 0.05
    x = rng.uniform(0.05, 1.0, (1, 6, 7))
    y = synth.simulate_rician(x, sigma, np.random.default_rng(4)).astype(np.float64)
    g = ops.rician_grad(x, y, sigma)
    h = 1e-6
    for _ in range(20):
        e = rng.standard_normal(x.shape)
        e /= np.linalg.norm(e)
        fd = (ops.rician_f(x + h * e, y, sigma) - ops.rician_f(x - h * e, y, sigma)) / (2 * h)
        an = float(np.sum(g * e))
        assert abs(fd - an) <= 1e-6 * (1.0 + abs(an))


def test_rician_special_cases():
    sigma = 0.1
    y = np.random.default_rng(0).uniform(0, 1, (1, 4, 4))
    assert np.array_equal(ops.rician_grad(np.zeros_like(y), y, sigma), np.zeros_like(y))   # B(0) = 0
    assert ops.rician_f(np.zeros_like(y), y, sigma) == 0.0                                  # log I0(0) = 0
    fid = ops.Fidelity("rician", y, sigma=sigma)
    with pytest.raises(NotImplementedError):
        fid.prox(y, 0.1)


def test_rician_config_is_stable_and_descends():
    """R1 reading: tau = 0.9 sigma^2 < 1/L_f. With beta = 0, lambda = 0 the iteration is gradient
    descent on f alone, so f decreases monotonically (descent lemma, P:972-type argument)."""
    cfg = configs.get("R1", batch=1, H=16, W=16)
    prob = synth.make_problem(cfg)
    fid = osolver.make_fidelities(cfg, prob)[0]
    x = prob["x0"][0].astype(np.float64)
    fprev = fid.value(x)
    for _ in range(30):
        x = x - cfg["tau"] * fid.grad(x)
        f = fid.value(x)
        assert f <= fprev + 1e-12
        fprev = f
