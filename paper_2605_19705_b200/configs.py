"""Frozen problem configurations C1..C5 (BASELINE.json configs, 1-based in list
order) with every reading of SURVEY.md §8(c)-6 spelled out. The same dicts feed
the input generator, the oracle tests and the CUDA path.

beta = 1 - alpha_paper (Eq. 4). ``step`` is "grad" (Alg. 1 l.8,
PAPER l.219) or "prox" (Alg. 2 l.7). ``max_iter`` counts operator
applications (reading Q2). ``tol`` is the relative residual threshold
||x^{k+1}-x^k||/||x^k|| <= tol (reading Q3).
"""
from __future__ import annotations

import copy

UNET32 = (32, 64, 128, 256)
UNET64 = (64, 128, 256, 512)

CONFIGS = {
    "C1": dict(name="C1 tiny deblur", seed_id=1, batch=1, C=1, H=32, W=32,
               net="tiny3", widths=(16, 0, 0, 0), identity_skip=True, act="softplus",
               op="blur", ksize=9, ksigma=1.6, kernel_per_image=False, sigma=0.01,
               blur_impl="direct", step="grad", lam=0.05, tau=1.0, beta=0.5,
               max_iter=100, tol=0.0, check_every=1, stop_rule="per_image",
               precision="fp32"),
    "C2": dict(name="C2 batched motion deblur", seed_id=2, batch=64, C=3, H=128, W=128,
               net="unet4", widths=UNET32, res_blocks=2, identity_skip=True, act="softplus",
               op="blur", ksize=15, kernel_per_image=True, walk_steps=20, sigma=0.02,
               blur_impl="direct", step="grad", lam=0.05, tau=1.0, beta=0.6,
               max_iter=200, tol=1e-4, check_every=1, stop_rule="per_image",
               precision="bf16"),
    "C3": dict(name="C3 random inpainting", seed_id=3, batch=32, C=3, H=256, W=256,
               net="unet4", widths=UNET32, res_blocks=2, identity_skip=True, act="softplus",
               op="inpaint", keep=0.5, sigma=0.01, step="prox", lam=0.05, tau=1.0, beta=0.7,
               max_iter=300, tol=1e-4, check_every=1, stop_rule="per_image",
               precision="bf16"),
    "C4": dict(name="C4 coded-diffraction phase retrieval", seed_id=4, batch=16, C=1, H=256, W=256,
               net="unet4", widths=UNET32, res_blocks=2, identity_skip=True, act="softplus",
               op="phase", n_phase=4, step="grad", lam=0.05, tau=0.5 / 17, beta=0.5,
               max_iter=300, tol=1e-4, check_every=1, stop_rule="per_image",
               precision="bf16"),
    "C5": dict(name="C5 large-batch deblur", seed_id=5, batch=512, C=3, H=512, W=512,
               net="unet4", widths=UNET64, res_blocks=2, identity_skip=True, act="softplus",
               op="blur", ksize=25, ksigma=3.0, kernel_per_image=False, sigma=0.01,
               blur_impl="fft", step="prox", lam=0.05, tau=1.0, beta=0.6,
               max_iter=200, tol=1e-4, check_every=10, stop_rule="global_max",
               precision="bf16"),
}


# Configurations of the §8(f) NEXT rows (not BASELINE configs; parity cases only).
# R1: Rician denoising (PAPER App. D.3.3), gradient variant only (no closed-form prox,
# P:1079). tau < 1/L with L_f <= 1/sigma^2 (B' <= 1/2 makes the Hessian of f at most 1/sigma^2):
# tau = 0.9 sigma^2; lambda scaled so that tau * lambda = 0.045 as in the blur/inpainting configs.
CONFIGS["R1"] = dict(name="R1 Rician denoising", seed_id=6, batch=4, C=1, H=128, W=128,
                     net="unet4", widths=UNET32, res_blocks=2, identity_skip=True, act="softplus",
                     op="rician", sigma=0.05, step="grad", lam=20.0, tau=0.9 * 0.05 ** 2, beta=0.5,
                     max_iter=100, tol=1e-4, check_every=1, stop_rule="per_image", precision="bf16")

# M1: compressed-sensing MRI (PAPER App. D.3.1; §4.1 x8 acceleration, sigma_y = 1/255
# P:1000), real magnitude image with zero phase, proximal variant (Alg. 2) with the
# closed-form prox (reading Q18). L_f = 1: tau = 1 is the blur/inpainting choice.
CONFIGS["M1"] = dict(name="M1 MRI x8", seed_id=7, batch=4, C=1, H=256, W=256,
                     net="unet4", widths=UNET32, res_blocks=2, identity_skip=True, act="softplus",
                     op="mri", accel=8, sigma=1.0 / 255, step="prox", lam=0.05, tau=1.0, beta=0.5,
                     max_iter=100, tol=1e-4, check_every=1, stop_rule="per_image", precision="bf16")


# Stress variants for parity: with the x0.1 init and lambda = 0.05 the
# regularizer term lam*grad g is ~1e-3 of grad f, so trajectory parity alone would not
# exercise the VJP. The stress variant uses init scale 0.3 and a larger lambda chosen so
# that ||lam grad g(x0)|| >= 0.1 ||grad f(0.9 x_true)|| while the oracle stays
# non-divergent over the parity horizon (checked in tests/test_oracle_configs.py).
STRESS = {
    "C1": dict(init_scale=0.3, lam=1.0),
    "C2": dict(init_scale=0.3, lam=0.1),
    "C3": dict(init_scale=0.3, lam=0.1),
    "C4": dict(init_scale=0.3, lam=5.0),
    "C5": dict(init_scale=0.3, lam=0.1),
    "R1": dict(init_scale=0.3, lam=200.0),
    "M1": dict(init_scale=0.3, lam=0.1),
}


def get(name: str, **overrides) -> dict:
    """A deep copy of config ``name`` with overrides applied (used for the
    reduced-size parity variants: fewer images, smaller H/W, fixed K)."""
    cfg = copy.deepcopy(CONFIGS[name])
    cfg.update(overrides)
    return cfg
