"""CPU pins of the oracle JFB gradient (oracle/jfb.py):
  - d/dtheta <v, grad g_theta(z)> against torch float64 double-backward (library pin: autograd of
    autograd on the same weights; neither product path uses torch for this);
  - the full JFB gradient (weights, lambda, tau) against central finite differences of the loss
    L = 1/2 ||T(x_hat) - x*||^2 (the definition), gradient and inpainting-prox variants.
"""
import numpy as np
import pytest

from oracle import jfb, nets
from oracle import solver as osolver
from paper_2605_19705_b200 import configs, synth

torch = pytest.importorskip("torch")


def _torch_net(net, C, widths):
    """The same U-Net / tiny net in torch (float64) with parameters from the oracle's dict."""
    F = torch.nn.functional
    Wt = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in net.W.items()}

    def sp(x):
        return F.softplus(x, beta=1.0, threshold=1e9)

    def U(x):
        x = x[None]
        if net.arch == "tiny3":
            a1 = sp(F.conv2d(x, Wt["c1"], padding=1))
            a2 = sp(F.conv2d(a1, Wt["c2"], padding=1))
            return F.conv2d(a2, Wt["c3"], padding=1)[0]
        t = F.conv2d(x, Wt["head"], padding=1)
        skips = {}
        for l in range(4):
            for r in range(net.res_blocks):
                t = t + F.conv2d(sp(F.conv2d(t, Wt[f"e{l}.{r}.A"], padding=1)), Wt[f"e{l}.{r}.B"], padding=1)
            if l < 3:
                skips[l] = t
                t = F.conv2d(t, Wt[f"down{l}"], stride=2)
        for l in (2, 1, 0):
            t = F.conv_transpose2d(t, Wt[f"up{l}"], stride=2) + skips[l]
            for r in range(net.res_blocks):
                t = t + F.conv2d(sp(F.conv2d(t, Wt[f"d{l}.{r}.A"], padding=1)), Wt[f"d{l}.{r}.B"], padding=1)
        return F.conv2d(t, Wt["tail"], padding=1)[0]
    return Wt, U


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C3", dict(batch=1, H=16, W=16, widths=(8, 8, 16, 16)))])
def test_phi_weight_grad_vs_torch_double_backward(name, kw):
    cfg = configs.get(name, init_scale=0.3, **kw)
    prob = synth.make_problem(cfg)
    net = osolver.make_net(cfg, prob["weights"])
    rng = np.random.default_rng(3)
    z = prob["x_true"][0].astype(np.float64)
    v = rng.standard_normal(z.shape)
    got = jfb.phi_weight_grad(net, z, v)
    Wt, U = _torch_net(net, cfg["C"], cfg["widths"])
    zt = torch.tensor(z, requires_grad=True)
    g = 0.5 * (U(zt) ** 2).sum()                         # g = 1/2 ||z - N(z)||^2 = 1/2 ||U(z)||^2
    (gg,) = torch.autograd.grad(g, zt, create_graph=True)
    phi = (gg * torch.tensor(v)).sum()
    want = torch.autograd.grad(phi, list(Wt.values()))
    for (k, _), w in zip(Wt.items(), want):
        ref = w.detach().numpy()
        assert np.linalg.norm(got[k] - ref) <= 1e-10 * max(np.linalg.norm(ref), 1e-300), k


def _loss(net, fid, z, xs, lam, tau, step):
    gg = net.grad_g(z)
    if step == "grad":
        T = z - tau * (fid.grad(z) + lam * gg)
    else:
        T = fid.prox(z - tau * lam * gg, tau)
    return 0.5 * float(np.sum((T - xs) ** 2))


@pytest.mark.parametrize("name,step,kw", [("C1", "grad", {}),
                                          ("C3", "prox", dict(batch=1, H=16, W=16, widths=(8, 8, 16, 16))),
                                          ("C3", "grad", dict(batch=1, H=16, W=16, widths=(8, 8, 16, 16)))])
def test_jfb_gradient_finite_differences(name, step, kw):
    cfg = configs.get(name, init_scale=0.3, step=step, **kw)
    prob = synth.make_problem(cfg)
    net = osolver.make_net(cfg, prob["weights"])
    fid = osolver.make_fidelities(cfg, prob)[0]
    z = (0.9 * prob["x_true"][0] + 0.05).astype(np.float64)         # a stand-in x_hat
    xs = prob["x_true"][0].astype(np.float64)
    lam, tau = 0.7, 0.6
    loss, dth, dlam, dtau, dbeta = jfb.jfb_grads(net, fid, z, xs, lam, tau, step)
    assert abs(loss - _loss(net, fid, z, xs, lam, tau, step)) <= 1e-12 * max(loss, 1.0)
    h = 1e-6
    assert abs((_loss(net, fid, z, xs, lam + h, tau, step) - _loss(net, fid, z, xs, lam - h, tau, step)) / (2 * h)
               - dlam) <= 1e-6 * (1 + abs(dlam))
    assert abs((_loss(net, fid, z, xs, lam, tau + h, step) - _loss(net, fid, z, xs, lam, tau - h, step)) / (2 * h)
               - dtau) <= 1e-6 * (1 + abs(dtau))
    assert dbeta == 0.0
    rng = np.random.default_rng(11)
    blob = np.asarray(prob["weights"], dtype=np.float64)
    for _ in range(4):
        d = rng.standard_normal(blob.shape)
        d /= np.linalg.norm(d)
        lp = _loss(osolver.make_net(cfg, blob + h * d), fid, z, xs, lam, tau, step)
        lm = _loss(osolver.make_net(cfg, blob - h * d), fid, z, xs, lam, tau, step)
        fd = (lp - lm) / (2 * h)
        assert abs(fd - float(dth @ d)) <= 1e-6 * (1 + abs(fd))
