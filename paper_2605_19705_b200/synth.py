"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This module holds no arithmetic of the i-DEQ iteration. It draws the random
quantities of a problem instance (ground-truth images, blur kernels, masks,
phase masks, noise, network weights) and simulates the acquisition
``y = A(x) + n`` (problem statement) so that both sides receive
the *same fp32-rounded* inputs. Any ``y`` is a valid input to the solver; the
simulation here only makes the data look like the paper's workloads.

Recipes follow SURVEY.md §8(c)-5 and §8(d)-2 (BASELINE.json configs); every
choice the paper leaves open is listed in DESIGN.md "Readings".
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "piecewise_smooth", "gaussian_kernel", "motion_kernel", "bernoulli_mask",
    "phase_masks", "he_normal_weights", "unet_weight_shapes", "tiny_weight_shapes",
    "simulate_blur", "simulate_inpaint", "simulate_phase", "simulate_rician", "cartesian_mask", "simulate_mri", "make_problem",
]


# --------------------------------------------------------------------------- images
def piecewise_smooth(rng: np.random.Generator, H: int, W: int, C: int) -> np.ndarray:
    """BASELINE.json C1: 6 random axis-aligned rectangles of uniform intensity in
    [0,1] (painted in order, later ones overwrite) plus 3 additive Gaussian blobs
    of sigma in [2,6] px, clipped to [0,1]. Returns float32 [C][H][W]."""
    img = np.zeros((H, W, C), dtype=np.float64)
    for _ in range(6):
        r = np.sort(rng.integers(0, H, size=2))
        c = np.sort(rng.integers(0, W, size=2))
        val = rng.uniform(0.0, 1.0, size=C)
        img[r[0]:r[1] + 1, c[0]:c[1] + 1, :] = val
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    for _ in range(3):
        cy = rng.uniform(0.0, H)
        cx = rng.uniform(0.0, W)
        s = rng.uniform(2.0, 6.0)
        amp = rng.uniform(0.0, 1.0, size=C)
        blob = np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2.0 * s * s))
        img += blob[:, :, None] * amp[None, None, :]
    img = np.clip(img, 0.0, 1.0)
    return np.ascontiguousarray(img.transpose(2, 0, 1)).astype(np.float32)


# --------------------------------------------------------------------------- operators' data
def gaussian_kernel(size: int, sigma: float) -> np.ndarray:
    """k[i,j] proportional to exp(-((i-c)^2+(j-c)^2)/(2 sigma^2)), sum 1 (BASELINE C1/C5)."""
    c = (size - 1) / 2.0
    i = np.arange(size, dtype=np.float64) - c
    k = np.exp(-(i[:, None] ** 2 + i[None, :] ** 2) / (2.0 * sigma * sigma))
    return (k / k.sum()).astype(np.float32)


def motion_kernel(rng: np.random.Generator, size: int = 15, steps: int = 20) -> np.ndarray:
    """BASELINE C2 random-walk motion blur: start at the centre, 20 steps of an
    8-neighbour walk (d != (0,0)), positions clipped to the grid, normalised."""
    k = np.zeros((size, size), dtype=np.float64)
    p = np.array([size // 2, size // 2])
    k[p[0], p[1]] += 1.0
    for _ in range(steps):
        while True:
            d = rng.integers(-1, 2, size=2)
            if d[0] != 0 or d[1] != 0:
                break
        p = np.clip(p + d, 0, size - 1)
        k[p[0], p[1]] += 1.0
    return (k / k.sum()).astype(np.float32)


def bernoulli_mask(rng: np.random.Generator, H: int, W: int, keep: float = 0.5) -> np.ndarray:
    """Per-image pixel mask, 1 = observed, shared by the channels (50% removed)."""
    return (rng.random((H, W)) < keep).astype(np.uint8)


def phase_masks(rng: np.random.Generator, J: int, H: int, W: int) -> np.ndarray:
    """D_j = exp(2 pi i U_j), U_j ~ U[0,1) (BASELINE C4). Returns float32 [J][H][W][2] (re, im)."""
    u = rng.random((J, H, W))
    d = np.exp(2j * np.pi * u)
    out = np.stack([d.real, d.imag], axis=-1).astype(np.float32)
    return np.ascontiguousarray(out)


# --------------------------------------------------------------------------- weights
def tiny_weight_shapes(C: int = 1, w: int = 16):
    """BASELINE C1 net: conv3x3 C->w, softplus, conv3x3 w->w, softplus, conv3x3 w->C."""
    return [("conv1", (w, C, 3, 3), C * 9), ("conv2", (w, w, 3, 3), w * 9),
            ("conv3", (C, w, 3, 3), w * 9)]


def unet_weight_shapes(C: int, widths, res_blocks: int = 2):
    """Blob order of include/ideq.h: head; per level l=0..3 the RB
    convs (A,B per block) then down_l (l<3); per decoder level l=2..0 up_l then
    the RB convs; tail. Conv layout [Cout][Cin][kh][kw]; up layout [Cin][Cout][2][2].
    Third field is fan_in for the He-normal init."""
    w = list(widths)
    shapes = [("head", (w[0], C, 3, 3), C * 9)]
    for l in range(4):
        for r in range(res_blocks):
            shapes.append((f"enc{l}.rb{r}.A", (w[l], w[l], 3, 3), w[l] * 9))
            shapes.append((f"enc{l}.rb{r}.B", (w[l], w[l], 3, 3), w[l] * 9))
        if l < 3:
            shapes.append((f"down{l}", (w[l + 1], w[l], 2, 2), w[l] * 4))
    for l in (2, 1, 0):
        shapes.append((f"up{l}", (w[l + 1], w[l], 2, 2), w[l + 1]))
        for r in range(res_blocks):
            shapes.append((f"dec{l}.rb{r}.A", (w[l], w[l], 3, 3), w[l] * 9))
            shapes.append((f"dec{l}.rb{r}.B", (w[l], w[l], 3, 3), w[l] * 9))
    shapes.append(("tail", (C, w[0], 3, 3), w[0] * 9))
    return shapes


def he_normal_weights(rng: np.random.Generator, shapes, scale: float = 0.1) -> np.ndarray:
    """W ~ N(0, (scale*sqrt(2/fan_in))^2), drawn tensor by tensor in blob order,
    C-order inside each tensor (BASELINE C1 "He-normal weights scaled 0.1, zero bias").
    Returns the flat float32 blob."""
    parts = []
    for _, shp, fan_in in shapes:
        std = scale * np.sqrt(2.0 / fan_in)
        parts.append(rng.normal(0.0, std, size=int(np.prod(shp))))
    return np.concatenate(parts).astype(np.float32)


# --------------------------------------------------------------------------- acquisition
def _circular_convolve(x: np.ndarray, k: np.ndarray) -> np.ndarray:
    """Acquisition-only helper: periodic true convolution of each channel of
    x [C][H][W] with the odd-sized kernel k whose tap ((s-1)/2,(s-1)/2) is the
    origin, evaluated through a zero-embedded kernel and a DFT (exact up to
    rounding)."""
    C, H, W = x.shape
    s = k.shape[0]
    c = (s - 1) // 2
    kp = np.zeros((H, W), dtype=np.float64)
    for i in range(s):
        for j in range(s):
            kp[(i - c) % H, (j - c) % W] += float(k[i, j])
    K = np.fft.fft2(kp)
    return np.real(np.fft.ifft2(np.fft.fft2(x.astype(np.float64), axes=(1, 2)) * K[None], axes=(1, 2)))


def simulate_blur(x: np.ndarray, k: np.ndarray, sigma: float, noise_rng) -> np.ndarray:
    y = _circular_convolve(x, k) + sigma * noise_rng.standard_normal(x.shape)
    return y.astype(np.float32)


def simulate_inpaint(x: np.ndarray, mask: np.ndarray, sigma: float, noise_rng) -> np.ndarray:
    """y = M (x + sigma n); unobserved pixels are exactly 0."""
    y = (x.astype(np.float64) + sigma * noise_rng.standard_normal(x.shape)) * mask[None].astype(np.float64)
    return y.astype(np.float32)


def simulate_phase(x: np.ndarray, D: np.ndarray, noise_rng) -> np.ndarray:
    """y_j = |FFT2(D_j x)|^2 (unitary DFT) + 0.01*mean(clean y) * n_j (BASELINE C4).
    x is [1][H][W]; D is [J][H][W][2]. Returns float32 [J][H][W]."""
    d = D[..., 0].astype(np.float64) + 1j * D[..., 1].astype(np.float64)
    u = np.fft.fft2(d * x[0][None].astype(np.float64), axes=(1, 2), norm="ortho")
    clean = np.abs(u) ** 2
    sig = 0.01 * clean.mean()
    y = clean + sig * noise_rng.standard_normal(clean.shape)
    return y.astype(np.float32)


def cartesian_mask(H: int, W: int, accel: int) -> np.ndarray:
    """Cartesian k-space mask (PAPER §4.1 "acceleration factor x8"; the paper's fastMRI mask
    generator is unstated): keep every phase-encode column kx with kx = 0 mod accel plus a fully
    sampled low-frequency band of max(4, W/32) columns around kx = 0. Both sets are closed under
    kx -> -kx, so the mask is Hermitian-symmetric (reading R7). Returns u8 [H][W]."""
    kx = np.arange(W)
    kxs = np.minimum(kx, W - kx)                    # |frequency| index
    band = max(4, W // 32)
    keep = (kx % accel == 0) | (kxs <= band // 2)
    return np.broadcast_to(keep[None, :], (H, W)).astype(np.uint8).copy()


def simulate_mri(x: np.ndarray, mask: np.ndarray, sigma: float, noise_rng) -> np.ndarray:
    """y = M F x + n, F the unitary 2-D DFT, n complex Gaussian (re, im ~ N(0, sigma^2)) on the
    sampled entries. x: [1][H][W]; returns float32 [H][W][2] (re, im)."""
    u = np.fft.fft2(x[0].astype(np.float64), norm="ortho")
    n = sigma * (noise_rng.standard_normal(u.shape) + 1j * noise_rng.standard_normal(u.shape))
    y = mask * (u + n)
    return np.stack([y.real, y.imag], axis=-1).astype(np.float32)


def simulate_rician(x: np.ndarray, sigma: float, noise_rng) -> np.ndarray:
    """Magnitude measurement y = sqrt((x + n_real)^2 + n_imag^2), n ~ N(0, sigma^2) iid
    (PAPER App. D.3.3). Returns float32, same shape as x."""
    nr = sigma * noise_rng.standard_normal(x.shape)
    ni = sigma * noise_rng.standard_normal(x.shape)
    return np.sqrt((x.astype(np.float64) + nr) ** 2 + ni ** 2).astype(np.float32)


# --------------------------------------------------------------------------- problems
def make_problem(cfg: dict, images=None) -> dict:
    """Build the inputs of one config (see configs.py). ``images`` selects a subset
    of image indices (default: all cfg['batch']). Every array is fp32 (u8 masks)
    and identical for the oracle and the GPU path."""
    N = cfg["batch"]
    idx = list(range(N)) if images is None else list(images)
    C, H, W = cfg["C"], cfg["H"], cfg["W"]
    cid = cfg["seed_id"]
    prob = {"cfg": cfg, "images": idx}

    # weights (BASELINE "random init with seed")
    wrng = np.random.default_rng([cid, 1000000])
    if cfg["net"] == "tiny3":
        shapes = tiny_weight_shapes(C, cfg["widths"][0])
    else:
        shapes = unet_weight_shapes(C, cfg["widths"], cfg.get("res_blocks", 2))
    prob["weights"] = he_normal_weights(wrng, shapes, cfg.get("init_scale", 0.1))
    prob["weight_shapes"] = [(n, s) for n, s, _ in shapes]

    xs, ys, ks, ms, x0s = [], [], [], [], []
    op = cfg["op"]
    if op == "phase":
        prob["phase_masks"] = phase_masks(np.random.default_rng([cid, 3]), cfg["n_phase"], H, W)
    if op == "mri":
        prob["kmask"] = cartesian_mask(H, W, cfg["accel"])
    if op == "blur" and not cfg.get("kernel_per_image", False):
        prob["kernel"] = gaussian_kernel(cfg["ksize"], cfg["ksigma"])
    for i in idx:
        if cid == 1:
            img_rng = np.random.default_rng(0)              # BASELINE C1 "seed 0"
            noise_rng = np.random.default_rng([1, 0, 1])
        else:
            img_rng = np.random.default_rng([cid, i])
            noise_rng = np.random.default_rng([cid, i, 1])
        x = piecewise_smooth(img_rng, H, W, C)
        xs.append(x)
        if op == "blur":
            if cfg.get("kernel_per_image", False):
                k = motion_kernel(np.random.default_rng([cid, i, 2]), cfg["ksize"], cfg.get("walk_steps", 20))
                ks.append(k)
            else:
                k = prob["kernel"]
            y = simulate_blur(x, k, cfg["sigma"], noise_rng)
            x0 = y.copy()
        elif op == "inpaint":
            m = bernoulli_mask(np.random.default_rng([cid, i, 2]), H, W, cfg.get("keep", 0.5))
            ms.append(m)
            y = simulate_inpaint(x, m, cfg["sigma"], noise_rng)
            x0 = y.copy()                                     # zero-filled start
        elif op == "rician":
            y = simulate_rician(x, cfg["sigma"], noise_rng)
            x0 = y.copy()
        elif op == "mri":
            y = simulate_mri(x, prob["kmask"], cfg["sigma"], noise_rng)
            # zero-filled start: x^0 = Re F^{-1} y (the standard MRI initialisation)
            x0 = np.real(np.fft.ifft2(y[..., 0].astype(np.float64) + 1j * y[..., 1], norm="ortho"))[None]
            x0 = x0.astype(np.float32)
        elif op == "phase":
            y = simulate_phase(x, prob["phase_masks"], noise_rng)
            x0 = np.full((C, H, W), np.sqrt(max(float(y.astype(np.float64).mean()), 0.0)), dtype=np.float32)
        else:
            raise ValueError(op)
        ys.append(y)
        x0s.append(x0)
    prob["x_true"] = np.stack(xs)
    prob["y"] = np.stack(ys)
    prob["x0"] = np.stack(x0s)
    if ks:
        prob["kernels"] = np.stack(ks)
    if ms:
        prob["masks"] = np.stack(ms)
    return prob
