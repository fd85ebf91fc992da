"""Oracle data-fidelity terms f, their gradients and proximal maps (fp64, one image).

Periodic blur (BASELINE C1/C2/C5; readings Q8, Q9):
  (Ax)[c,m,n]  = sum_{i,j} k[i,j] x[c, (m-i+kc) mod H, (n-j+kc) mod W]   true convolution
  (A^T r)      = sum_{i,j} k[i,j] r[c, (m+i-kc) mod H, (n+j-kc) mod W]   correlation
  f = 1/2 ||Ax - y||^2,  grad f = A^T(Ax - y)         (by analogy with P:964)
  prox_{tau f}(v) = argmin_x 1/2||Ax-y||^2 + ||x-v||^2/(2 tau)
                  = (I + tau A^T A)^{-1}(v + tau A^T y)
                  = F^{-1}[ F(v + tau A^T y) / (1 + tau |K^|^2) ]   (A circulant)
Inpainting (PAPER App. D.3.2):
  f = 1/2 ||Mx - y||^2, grad f = M^T(Mx - y),
  prox_{tau f}(v) = (tau M y + v) / (tau M + 1) componentwise.
Coded-diffraction phase retrieval (BASELINE C4; reading Q7, Q14):
  f = 1/2 sum_j || |F(D_j x)|^2 - y_j ||^2, F the unitary 2-D DFT,
  grad f = sum_j 2 Re( conj(D_j) F^{-1}[ (|u_j|^2 - y_j) u_j ] ),  u_j = F(D_j x).
Compressed-sensing MRI (PAPER App. D.3.1; readings Q18, R7):
  x real (zero phase), y complex k-space, F the unitary 2-D DFT, M a binary mask:
  f = 1/2 ||M F x - y||^2, grad f = Re F^{-1} M^T (M F x - y),
  prox_{tau f}(v) = Re F^{-1}[ (F v + tau M y) / (1 + tau M) ] (P:985 read in k-space, Q18).
Rician denoising (PAPER App. D.3.3):
  f = sum x^2 / (2 sigma^2) - log I0(x y / sigma^2),
  grad f = x / sigma^2 - (y / sigma^2) B(x y / sigma^2),  B = I1 / I0;  no closed-form prox.
  I0, I1 via the exponentially scaled library routines scipy.special.i0e / i1e (library step).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


# --------------------------------------------------------------------------- blur
def blur_A(x, k):
    """Direct periodic true convolution, written as the defining sum of shifted copies."""
    s = k.shape[0]
    kc = (s - 1) // 2
    out = np.zeros_like(x, dtype=np.float64)
    for i in range(s):
        for j in range(s):
            # np.roll(x, d)[m] = x[m - d]  =>  d = i - kc gives x[m - i + kc]
            out += float(k[i, j]) * np.roll(x, (i - kc, j - kc), axis=(-2, -1))
    return out


def blur_AT(r, k):
    """Adjoint of blur_A: correlation r[m + i - kc]."""
    s = k.shape[0]
    kc = (s - 1) // 2
    out = np.zeros_like(r, dtype=np.float64)
    for i in range(s):
        for j in range(s):
            out += float(k[i, j]) * np.roll(r, (-(i - kc), -(j - kc)), axis=(-2, -1))
    return out


def blur_f(x, y, k):
    r = blur_A(x, k) - y
    return 0.5 * float(np.sum(r * r))


def blur_grad(x, y, k):
    """grad f = A^T(Ax - y)."""
    return blur_AT(blur_A(x, k) - y, k)


def blur_transfer(k, H, W):
    """K^ = unnormalised 2-D DFT of k zero-embedded in H x W with tap (kc,kc) at (0,0)."""
    s = k.shape[0]
    kc = (s - 1) // 2
    kp = np.zeros((H, W))
    for i in range(s):
        for j in range(s):
            kp[(i - kc) % H, (j - kc) % W] += float(k[i, j])
    return np.fft.fft2(kp)


def blur_prox(v, y, k, tau):
    """prox_{tau f}(v) = F^{-1}[ F(v + tau A^T y) / (1 + tau |K^|^2) ] (per channel)."""
    H, W = v.shape[-2:]
    K = blur_transfer(k, H, W)
    rhs = v + tau * blur_AT(y, k)
    return np.real(np.fft.ifft2(np.fft.fft2(rhs, axes=(-2, -1)) / (1.0 + tau * np.abs(K) ** 2),
                                axes=(-2, -1)))


# --------------------------------------------------------------------------- inpainting
def inpaint_f(x, y, m):
    r = m * x - y
    return 0.5 * float(np.sum(r * r))


def inpaint_grad(x, y, m):
    """grad f = M^T (M x - y); M diagonal, shared by the channels."""
    return m * (m * x - y)


def inpaint_prox(v, y, m, tau):
    """(tau M y + v) / (tau M + 1), componentwise."""
    return (tau * m * y + v) / (tau * m + 1.0)


# --------------------------------------------------------------------------- phase retrieval
def _dft(a):
    return np.fft.fft2(a, axes=(-2, -1), norm="ortho")


def _idft(a):
    return np.fft.ifft2(a, axes=(-2, -1), norm="ortho")


def phase_f(x, y, D):
    """x: [1][H][W]; y: [J][H][W]; D: [J][H][W] complex."""
    u = _dft(D * x[0][None])
    r = np.abs(u) ** 2 - y
    return 0.5 * float(np.sum(r * r))


def phase_grad(x, y, D):
    u = _dft(D * x[0][None])
    w = (np.abs(u) ** 2 - y) * u
    g = np.sum(2.0 * np.real(np.conj(D) * _idft(w)), axis=0)
    return g[None]


# --------------------------------------------------------------------------- MRI
def mri_f(x, y, m):
    """x: [1][H][W] real; y: [H][W] complex; m: [H][W] in {0, 1}."""
    r = m * _dft(x[0]) - y
    return 0.5 * float(np.sum(np.abs(r) ** 2))


def mri_grad(x, y, m):
    """Re F^{-1} M^T (M F x - y); F^{-1} = F^H for the unitary DFT."""
    return np.real(_idft(m * (m * _dft(x[0]) - y)))[None]


def mri_prox(v, y, m, tau):
    """Re F^{-1}[(F v + tau M y) / (1 + tau M)] (reading Q18)."""
    return np.real(_idft((_dft(v[0]) + tau * m * y) / (1.0 + tau * m)))[None]


# --------------------------------------------------------------------------- Rician
def bessel_ratio(t):
    """B(t) = I1(t) / I0(t) = i1e(t) / i0e(t): the e^{-t} scalings cancel, no overflow."""
    from scipy.special import i0e, i1e
    t = np.asarray(t, dtype=np.float64)
    return i1e(t) / i0e(t)


def log_i0(t):
    """log I0(t) = t + log i0e(t) for t >= 0 (I0 is even)."""
    from scipy.special import i0e
    t = np.abs(np.asarray(t, dtype=np.float64))
    return t + np.log(i0e(t))


def rician_f(x, y, sigma):
    """f = sum x^2 / (2 sigma^2) - log I0(x y / sigma^2)."""
    s2 = sigma * sigma
    return float(np.sum(x * x / (2.0 * s2) - log_i0(x * y / s2)))


def rician_grad(x, y, sigma):
    """grad f = x / sigma^2 - (y / sigma^2) B(x y / sigma^2). B is odd: B(-t) = -B(t)."""
    s2 = sigma * sigma
    t = x * y / s2
    return x / s2 - (y / s2) * np.sign(t) * bessel_ratio(np.abs(t))


# --------------------------------------------------------------------------- dispatch
class Fidelity:
    """f(., y) for one image: value, gradient, prox (None when not closed form)."""

    def __init__(self, kind, y, kernel=None, mask=None, phase=None, sigma=None):
        self.kind = kind
        self.sigma = sigma
        if kind == "mri":  # y: [H][W][2] (re, im) -> complex; mask: [H][W] k-space
            y = np.asarray(y, dtype=np.float64)
            self.y = y[..., 0] + 1j * y[..., 1]
            self.km = np.asarray(mask, dtype=np.float64)
            return
        self.y = np.asarray(y, dtype=np.float64)
        self.k = None if kernel is None else np.asarray(kernel, dtype=np.float64)
        self.m = None if mask is None else np.asarray(mask, dtype=np.float64)[None]
        if phase is not None:
            phase = np.asarray(phase, dtype=np.float64)
            self.D = phase[..., 0] + 1j * phase[..., 1]

    def value(self, x):
        if self.kind == "blur":
            return blur_f(x, self.y, self.k)
        if self.kind == "inpaint":
            return inpaint_f(x, self.y, self.m)
        if self.kind == "rician":
            return rician_f(x, self.y, self.sigma)
        if self.kind == "mri":
            return mri_f(x, self.y, self.km)
        return phase_f(x, self.y, self.D)

    def grad(self, x):
        if self.kind == "blur":
            return blur_grad(x, self.y, self.k)
        if self.kind == "inpaint":
            return inpaint_grad(x, self.y, self.m)
        if self.kind == "rician":
            return rician_grad(x, self.y, self.sigma)
        if self.kind == "mri":
            return mri_grad(x, self.y, self.km)
        return phase_grad(x, self.y, self.D)

    def prox(self, v, tau):
        if self.kind == "blur":
            return blur_prox(v, self.y, self.k, tau)
        if self.kind == "inpaint":
            return inpaint_prox(v, self.y, self.m, tau)
        if self.kind == "mri":
            return mri_prox(v, self.y, self.km, tau)
        raise NotImplementedError("no closed-form prox for phase retrieval / Rician (P:1079)")
