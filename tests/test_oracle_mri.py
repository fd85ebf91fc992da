"""CPU pins of the oracle's compressed-sensing MRI fidelity (PAPER App. D.3.1; SURVEY
§8(f) NEXT-3; readings Q18, R7): finite differences of f, the Lipschitz certificate L = 1,
prox optimality x + tau grad f(x) = v (exact for the Hermitian-symmetric Cartesian mask, which
makes the k-space reading of P:985 the prox over REAL images), the all-ones-mask closed form, and
the zero gradient at the noise-free truth."""
import numpy as np
import pytest

from oracle import operators as ops
from paper_2605_19705_b200 import synth


def _problem(H=32, W=32, accel=4, sigma=0.01, seed=0):
    rng = np.random.default_rng(seed)
    x = synth.piecewise_smooth(rng, H, W, 1).astype(np.float64)
    m = synth.cartesian_mask(H, W, accel)
    y = synth.simulate_mri(x, m, sigma, np.random.default_rng(seed + 1))
    return x, m, ops.Fidelity("mri", y, mask=m)


def test_cartesian_mask_hermitian_and_rate():
    for (H, W, R) in [(32, 32, 4), (64, 128, 8), (256, 256, 8)]:
        m = synth.cartesian_mask(H, W, R).astype(np.float64)
        flip = np.roll(m[::-1, ::-1], (1, 1), axis=(0, 1))          # m[-ky, -kx]
        assert np.array_equal(m, flip)
        assert m[:, 0].all() and m[:, W // R].all()
        assert 1.0 / R <= m.mean() <= 1.0 / R + (max(4, W // 32) + 2) / W


def test_mri_gradient_finite_differences():
    x, m, fid = _problem()
    rng = np.random.default_rng(5)
    g = fid.grad(x)
    h = 1e-6
    for _ in range(20):
        e = rng.standard_normal(x.shape)
        e /= np.linalg.norm(e)
        fd = (fid.value(x + h * e) - fid.value(x - h * e)) / (2 * h)
        an = float(np.sum(g * e))
        assert abs(fd - an) <= 1e-7 * (1.0 + abs(an))


def test_mri_lipschitz_one():
    x, m, fid = _problem()
    rng = np.random.default_rng(6)
    for _ in range(10):
        a, b = rng.standard_normal(x.shape), rng.standard_normal(x.shape)
        assert np.linalg.norm(fid.grad(a) - fid.grad(b)) <= np.linalg.norm(a - b) * (1 + 1e-12)


@pytest.mark.parametrize("tau", [0.3, 1.0, 5.0])
def test_mri_prox_optimality(tau):
    x, m, fid = _problem()
    v = np.random.default_rng(7).standard_normal(x.shape)
    p = fid.prox(v, tau)
    assert np.linalg.norm(p + tau * fid.grad(p) - v) <= 1e-12 * np.linalg.norm(v)


def test_mri_all_ones_mask_and_truth():
    H = W = 16
    rng = np.random.default_rng(8)
    x = rng.uniform(0, 1, (1, H, W))
    ones = np.ones((H, W), dtype=np.uint8)
    u = np.fft.fft2(x[0], norm="ortho")                                         # noise-free, full, fp64
    yc = np.stack([u.real, u.imag], axis=-1)
    fid = ops.Fidelity("mri", yc, mask=ones)
    assert np.max(np.abs(fid.grad(x))) <= 1e-12                                 # grad f(x_true) = 0
    v = rng.standard_normal(x.shape)
    tau = 0.7
    want = (v + tau * x) / (1.0 + tau)                                          # F^{-1} y = x
    assert np.allclose(fid.prox(v, tau), want, rtol=0, atol=1e-12)
