"""GPU-vs-oracle parity at BASELINE.json's full per-GPU sizes ("Oracle cost").

Each case runs the CUDA path on the WHOLE per-GPU batch of a config in bf16 (the launch
configuration bench.py times for C3: 32 x 3 x 256 x 256, U-Net-32, inpainting prox) and
checks SAMPLED images against the fp64 oracle run one image at a time: the first and the
last image of the batch (so the last M tile and the batch stride are exercised).

Bars (north_star): bf16 reconstruction PSNR within 0.05 dB of the oracle's; the component
grad g within the documented bf16 bound (3e-2 relative). The fp32 FFMA mode is checked at
the full C3 size against the 1e-4 iterate bar. C5 runs at its per-GPU shard (64 of 512
images at P = 8) with the sampled image for one iteration (the oracle needs ~1 min/image-iter).
"""
import numpy as np
import pytest

from oracle import solver as osolver
from paper_2605_19705_b200 import configs, synth
from tests.gpu_util import psnr, rel_l2, torch_cuda

pytestmark = pytest.mark.gpu

FULL = {"C2": dict(), "C3": dict(), "C4": dict(), "C5": dict(batch=64)}
K_FULL = {"C2": 3, "C3": 3, "C4": 3, "C5": 1}


def _dev(torch, a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _samples(cfg):
    n = cfg["batch"]
    return [n - 1] if cfg["H"] >= 512 else [0, n - 1]


def _gpu_solve(cfg, prob, precision, K, lam=None):
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    s = ideq.Solver(cfg, prob["weights"], precision=precision, max_batch=cfg["batch"])
    s.set_operator(prob)
    xd = _dev(torch, prob["x0"])
    st, code, _ = s.solve(_dev(torch, prob["y"]), xd, s.params(lam=lam, max_iter=K, tol=0.0))
    x = xd.cpu().numpy()
    s.close()
    return st, x


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_fullsize_bf16_trajectory_sampled(name):
    """Whole batch on the GPU (bf16, tcgen05), oracle on sampled images: PSNR gap <= 0.05 dB,
    iterate rel-L2 and final residual close (the regularizer is a small part of the step)."""
    cfg = configs.get(name, **FULL[name])
    K = K_FULL[name]
    prob = synth.make_problem(cfg)
    st, x = _gpu_solve(cfg, prob, "bf16", K)
    assert (st["iters"] == K).all() and (st["status"] == 1).all()
    assert np.isfinite(x).all()
    for i in _samples(cfg):
        sub = synth.make_problem(cfg, images=[i])
        assert np.array_equal(sub["y"][0], prob["y"][i])
        orc = osolver.solve_config(cfg, sub, max_iter=K, tol=0.0)
        d = abs(psnr(x[i], prob["x_true"][i]) - psnr(orc["x"][0], prob["x_true"][i]))
        assert d <= 0.05, (i, d)
        assert rel_l2(x[i], orc["x"][0]) <= 2e-3, i
        assert abs(st["residual"][i] - orc["residual"][0]) <= 2e-3 * max(orc["residual"][0], 1e-3), i


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_fullsize_bf16_grad_g_sampled(name):
    """grad g(z) = (I - J_N)^T (z - N(z)) (Eq. 2) over the full batch; sampled images vs the
    oracle at the stress init (x0.3) so the softplus nonlinearity is exercised."""
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    cfg = configs.get(name, init_scale=configs.STRESS[name]["init_scale"], **FULL[name])
    prob = synth.make_problem(cfg)
    s = ideq.Solver(cfg, prob["weights"], precision="bf16", max_batch=cfg["batch"])
    s.set_operator(prob)
    z = prob["x_true"].astype(np.float32)
    zd = _dev(torch, z)
    g = torch.zeros_like(zd)
    u = torch.zeros_like(zd)
    s.grad_g(zd, g, u)
    gh, uh = g.cpu().numpy(), u.cpu().numpy()
    s.close()
    net = osolver.make_net(cfg, prob["weights"])
    for i in _samples(cfg):
        zi = z[i].astype(np.float64)
        assert rel_l2(gh[i], net.grad_g(zi)) <= 3e-2, i
        assert rel_l2(uh[i], net.N(zi) - zi) <= 3e-2, i


def test_fullsize_c3_fp32_trajectory_sampled():
    """fp32 (FFMA) mode at the full C3 size with the stress lambda: iterates within 1e-4
    relative L2 and residuals within 1e-6 of the oracle (north_star)."""
    name = "C3"
    cfg = configs.get(name, init_scale=configs.STRESS[name]["init_scale"])
    lam = configs.STRESS[name]["lam"]
    K = 2
    prob = synth.make_problem(cfg)
    st, x = _gpu_solve(cfg, prob, "fp32", K, lam=lam)
    for i in _samples(cfg):
        sub = synth.make_problem(cfg, images=[i])
        orc = osolver.solve_config(cfg, sub, max_iter=K, tol=0.0, lam=lam)
        assert rel_l2(x[i], orc["x"][0]) <= 1e-4, i
        assert abs(st["residual"][i] - orc["residual"][0]) <= 1e-6, i
