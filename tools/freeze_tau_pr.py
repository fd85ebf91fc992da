"""Freeze the phase-retrieval step size tau_PR (reading Q12 in DESIGN.md).

tau_PR = 0.5 / L^, where L^ is 30 steps of fp64 power iteration on the
finite-difference Hessian-vector product of f at x^0 (image 0), rounded down to 2
significant digits. Calls only oracle/ and the input generator; prints the values that
configs.py / the tests freeze.

    python tools/freeze_tau_pr.py
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import solver  # noqa: E402
from paper_2605_19705_b200 import configs, synth  # noqa: E402


def lipschitz_estimate(cfg, iters=30, h=1e-6):
    prob = synth.make_problem(cfg, images=[0])
    fid = solver.make_fidelities(cfg, prob)[0]
    x0 = prob["x0"][0].astype(np.float64)
    v = np.random.default_rng(0).standard_normal(x0.shape)
    v /= np.linalg.norm(v)
    lam = 0.0
    for _ in range(iters):
        hv = (fid.grad(x0 + h * v) - fid.grad(x0 - h * v)) / (2 * h)
        lam = float(np.linalg.norm(hv))
        v = hv / lam
    return lam


def round_down_2sig(v):
    e = math.floor(math.log10(v))
    return math.floor(v / 10 ** (e - 1)) * 10 ** (e - 1)


if __name__ == "__main__":
    for label, cfg in [("C4", configs.get("C4", tau=1.0)),
                       ("C4-mini (tests)", configs.get("C4", batch=2, H=64, W=32, tau=1.0))]:
        L = lipschitz_estimate(cfg)
        Lr = round_down_2sig(L)
        print(f"{label}: L^ = {L:.6g} -> {Lr:.2g}, tau_PR = 0.5 / L^ = {0.5 / Lr:.6g}")
