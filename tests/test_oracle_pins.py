"""Pins of the fp64 oracle against things other than itself.

Each test names the pin it implements and the passage it follows. These run on CPU.
"""
import json
import os

import numpy as np
import pytest

from oracle import nets, operators, solver
from paper_2605_19705_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")


def _unet(C=3, widths=(8, 8, 16, 16), scale=1.0, seed=0, skip=True, act="softplus"):
    shapes = synth.unet_weight_shapes(C, widths)
    blob = synth.he_normal_weights(np.random.default_rng(seed), shapes, scale)
    return nets.Net("unet4", blob, C, widths, skip, act), blob


def _tiny(C=1, w=16, scale=1.0, seed=0, skip=True, act="softplus"):
    shapes = synth.tiny_weight_shapes(C, w)
    blob = synth.he_normal_weights(np.random.default_rng(seed), shapes, scale)
    return nets.Net("tiny3", blob, C, (w, 0, 0, 0), skip, act), blob


# ----------------------------------------------------------------------------- P1
@pytest.mark.parametrize("kind", ["tiny", "tiny_noskip", "unet", "unet_linear"])
def test_P1_grad_g_central_differences(kind):
    """P1: <grad g(x), d> vs (g(x+hd) - g(x-hd)) / 2h along random unit d."""
    rng = np.random.default_rng(1)
    if kind.startswith("tiny"):
        net, _ = _tiny(skip=(kind == "tiny"))
        x = rng.uniform(0, 1, (1, 8, 8))
    else:
        net, _ = _unet(act="identity" if kind == "unet_linear" else "softplus")
        x = rng.uniform(0, 1, (3, 16, 16))
    gr = net.grad_g(x)
    h = 1e-5
    for _ in range(20 if kind.startswith("tiny") else 6):
        d = rng.standard_normal(x.shape)
        d /= np.linalg.norm(d)
        fd = (net.g(x + h * d) - net.g(x - h * d)) / (2 * h)
        an = float(np.sum(gr * d))
        assert abs(fd - an) <= 1e-6 * (1 + abs(an)), (fd, an)


# ----------------------------------------------------------------------------- P2
def _torch_unet_N(torch, x, W, widths, act_sp=True):
    F = torch.nn.functional

    def sp(t):
        return torch.clamp(t, min=0) + torch.log1p(torch.exp(-torch.abs(t))) if act_sp else t
    t = F.conv2d(x, W["head"], padding=1)
    skips = {}
    for l in range(4):
        for r in range(2):
            t = t + F.conv2d(sp(F.conv2d(t, W[f"e{l}.{r}.A"], padding=1)), W[f"e{l}.{r}.B"], padding=1)
        if l < 3:
            skips[l] = t
            t = F.conv2d(t, W[f"down{l}"], stride=2)
    for l in (2, 1, 0):
        t = F.conv_transpose2d(t, W[f"up{l}"], stride=2) + skips[l]
        for r in range(2):
            t = t + F.conv2d(sp(F.conv2d(t, W[f"d{l}.{r}.A"], padding=1)), W[f"d{l}.{r}.B"], padding=1)
    return x + F.conv2d(t, W["tail"], padding=1)


def test_P2_unet_vs_torch_float64_autograd():
    """P2: library pin -- torch CPU float64 conv2d / conv_transpose2d + autograd on the
    same weights give N(z) and grad g(z) to 1e-12 relative."""
    torch = pytest.importorskip("torch")
    widths = (8, 16, 16, 32)
    net, blob = _unet(widths=widths)
    rng = np.random.default_rng(2)
    z = rng.uniform(0, 1, (3, 32, 32))
    W = {k: torch.tensor(v) for k, v in nets.unpack_unet(blob, 3, widths).items()}
    xt = torch.tensor(z[None], requires_grad=True)
    n = _torch_unet_N(torch, xt, W, widths)
    g = 0.5 * torch.sum((xt - n) ** 2)
    g.backward()
    n_or = net.N(z)
    gg_or = net.grad_g(z)
    n_t = n.detach().numpy()[0]
    gg_t = xt.grad.numpy()[0]
    assert np.linalg.norm(n_or - n_t) <= 1e-12 * np.linalg.norm(n_t)
    assert np.linalg.norm(gg_or - gg_t) <= 1e-12 * np.linalg.norm(gg_t)


def test_P2_tiny_vs_torch_float64_autograd():
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    net, blob = _tiny(w=16)
    W = {k: torch.tensor(v) for k, v in nets.unpack_tiny(blob, 1, 16).items()}
    z = np.random.default_rng(3).uniform(0, 1, (1, 32, 32))
    xt = torch.tensor(z[None], requires_grad=True)

    def sp(t):
        return torch.clamp(t, min=0) + torch.log1p(torch.exp(-torch.abs(t)))
    n = xt + F.conv2d(sp(F.conv2d(sp(F.conv2d(xt, W["c1"], padding=1)), W["c2"], padding=1)), W["c3"], padding=1)
    (0.5 * torch.sum((xt - n) ** 2)).backward()
    gg = net.grad_g(z)
    assert np.linalg.norm(gg - xt.grad.numpy()[0]) <= 1e-12 * np.linalg.norm(gg)


# ----------------------------------------------------------------------------- P3
def test_P3_special_cases():
    """P3: zero-output net without skip => grad g = x; identity net => grad g = 0."""
    x = np.random.default_rng(4).uniform(0, 1, (3, 16, 16))
    net, blob = _unet(scale=0.0, skip=False)
    assert np.array_equal(net.grad_g(x), x)
    assert net.g(x) == pytest.approx(0.5 * np.sum(x * x), rel=1e-15)
    net, _ = _unet(scale=0.0, skip=True)
    assert np.array_equal(net.grad_g(x), np.zeros_like(x))
    assert net.g(x) == 0.0
    t, _ = _tiny(scale=0.0, skip=False)
    x1 = x[:1]
    assert np.array_equal(t.grad_g(x1), x1)


# ----------------------------------------------------------------------------- P4
def _dense(op, shape):
    n = int(np.prod(shape))
    M = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        M[:, j] = op(e.reshape(shape)).ravel()
    return M


@pytest.mark.parametrize("op", ["blur", "inpaint"])
@pytest.mark.parametrize("beta,step", [(0.0, "grad"), (0.5, "grad"), (0.0, "prox"), (0.5, "prox")])
def test_P4_linear_net_fixed_point_dense_solve(op, beta, step):
    """P4: linear N (act = identity, no skip) => g = 1/2||(I-W)x||^2 and the fixed point solves
    (A^T A + lam (I-W)^T (I-W)) x = A^T y, assembled from forward applications only
    (stationarity of Eq. 1 at a fixed point)."""
    H = Wd = 16
    shape = (1, H, Wd)
    net, _ = _tiny(scale=0.3, skip=False, act="identity")
    rng = np.random.default_rng(5)
    y = rng.uniform(0, 1, shape)
    if op == "blur":
        k = synth.gaussian_kernel(9, 1.6).astype(np.float64)
        A = _dense(lambda v: operators.blur_A(v, k), shape)
        fid = operators.Fidelity("blur", y, kernel=k)
    else:
        m = synth.bernoulli_mask(rng, H, Wd)
        A = np.diag(np.broadcast_to(m[None], shape).ravel().astype(np.float64))
        y = y * m[None]
        fid = operators.Fidelity("inpaint", y, mask=m)
    Wm = _dense(lambda v: net.U_forward(v)[0], shape)       # N = U, linear
    I = np.eye(Wm.shape[0])
    lam = 0.5
    Q = A.T @ A + lam * (I - Wm).T @ (I - Wm)
    xs = np.linalg.solve(Q, A.T @ y.ravel()).reshape(shape)
    tau = 0.8 if step == "grad" else 1.0
    out = solver.solve(net, [fid], y[None], lam, tau, beta, 3000, 1e-13, step)
    err = np.linalg.norm(out["x"][0] - xs) / np.linalg.norm(xs)
    assert err <= 1e-8, err


# ----------------------------------------------------------------------------- P5
def _red_loop(net, fid, x0, lam, tau, K):
    """Eq. 3 written separately: x - tau(grad f + lam (x - D(x))) with
    x - D(x) = grad g(x) (Eq. 2, D = Id - grad g). The D-form itself is checked to 1e-13."""
    x = x0.copy()
    xs = []
    for _ in range(K):
        gg = net.grad_g(x)
        D = x - gg
        x_d = x - tau * (fid.grad(x) + lam * (x - D))
        x = x - tau * (fid.grad(x) + lam * gg)
        assert np.abs(x_d - x).max() <= 1e-13 * (1 + np.abs(x).max())
        xs.append(x)
    return xs


def _redp_loop(net, fid, x0, lam, tau, K):
    """RED-P: x^{k+1} = prox_{tau f}(x^k - tau lam grad g(x^k))."""
    x = x0.copy()
    xs = []
    for _ in range(K):
        x = fid.prox(x - tau * lam * net.grad_g(x), tau)
        xs.append(x)
    return xs


@pytest.mark.parametrize("variant", ["red", "redp"])
def test_P5_beta0_reduces_to_red_bitwise(variant):
    """P5: beta = 0 (alpha = 1) reproduces RED / RED-P = ELDER's iteration bit for bit."""
    net, _ = _tiny(scale=1.0)
    rng = np.random.default_rng(6)
    H = 16
    x0 = rng.uniform(0, 1, (1, H, H))
    if variant == "red":
        fid = operators.Fidelity("blur", x0, kernel=synth.gaussian_kernel(9, 1.6))
        ref = _red_loop(net, fid, x0, 0.2, 0.9, 50)
        step = "grad"
    else:
        m = synth.bernoulli_mask(rng, H, H)
        fid = operators.Fidelity("inpaint", x0 * m[None], mask=m)
        ref = _redp_loop(net, fid, x0, 0.2, 1.0, 50)
        step = "prox"
    out = solver.solve(net, [fid], x0[None], 0.2, 0.9 if variant == "red" else 1.0, 0.0, 50, 0.0, step)
    # The z = x + 0*(x - x_prev) = x identity makes every iterate bit-identical.
    assert np.array_equal(out["x"][0], ref[-1])
    x = x0.copy()
    xp = x0.copy()
    for k in range(50):
        xn = solver.ideq_step(x, xp, net, fid, 0.2, 0.9 if variant == "red" else 1.0, 0.0, step)
        assert np.array_equal(xn, ref[k])
        xp, x = x, xn


# ----------------------------------------------------------------------------- P6
def _naive_dft2(a):
    H, W = a.shape
    m = np.arange(H)
    n = np.arange(W)
    FH = np.exp(-2j * np.pi * np.outer(m, m) / H)
    FW = np.exp(-2j * np.pi * np.outer(n, n) / W)
    return FH @ a @ FW.T


def test_P6_fft_primitive_vs_naive_dft():
    """P6(i): the FFT primitive vs the O(N^2) DFT definition; round trip and Parseval."""
    rng = np.random.default_rng(7)
    for H, W in [(8, 8), (16, 16), (8, 12)]:
        a = rng.standard_normal((H, W)) + 1j * rng.standard_normal((H, W))
        assert np.abs(np.fft.fft2(a) - _naive_dft2(a)).max() <= 1e-12 * np.abs(_naive_dft2(a)).max()
        u = operators._dft(a)
        assert abs(np.linalg.norm(u) - np.linalg.norm(a)) <= 1e-12 * np.linalg.norm(a)
        assert np.abs(operators._idft(u) - a).max() <= 1e-12


@pytest.mark.parametrize("ks,sig,H,W", [(9, 1.6, 32, 32), (25, 3.0, 64, 48)])
def test_P6_fft_blur_vs_direct(ks, sig, H, W):
    """P6(ii): the transfer-function form K^ F(x) equals the direct periodic convolution."""
    k = synth.gaussian_kernel(ks, sig).astype(np.float64)
    x = np.random.default_rng(8).uniform(0, 1, (3, H, W))
    K = operators.blur_transfer(k, H, W)
    via_fft = np.real(np.fft.ifft2(np.fft.fft2(x, axes=(1, 2)) * K, axes=(1, 2)))
    assert np.abs(via_fft - operators.blur_A(x, k)).max() <= 1e-12


def test_P6_motion_kernel_direct_blur_brute_force():
    """P6(ii) on an asymmetric kernel: blur_A and blur_AT vs brute-force index loops of the
    definitions (reading Q8) and the adjoint identity <Ax, r> = <x, A^T r>."""
    rng = np.random.default_rng(9)
    k = synth.motion_kernel(rng, 15).astype(np.float64)
    H, W = 12, 10
    x = rng.standard_normal((1, H, W))
    r = rng.standard_normal((1, H, W))
    kc = 7
    bf = np.zeros((1, H, W))
    for m in range(H):
        for n in range(W):
            s = 0.0
            for i in range(15):
                for j in range(15):
                    s += k[i, j] * x[0, (m - i + kc) % H, (n - j + kc) % W]
            bf[0, m, n] = s
    assert np.abs(bf - operators.blur_A(x, k)).max() <= 1e-13
    lhs = float(np.sum(operators.blur_A(x, k) * r))
    rhs = float(np.sum(x * operators.blur_AT(r, k)))
    assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)


# ----------------------------------------------------------------------------- P7
@pytest.mark.parametrize("tau", [1.0, 0.3])
def test_P7_prox_optimality(tau):
    """P7: x + tau grad f(x) = v at x = prox_{tau f}(v), with the direct operators."""
    rng = np.random.default_rng(10)
    H, W = 24, 20
    v = rng.standard_normal((3, H, W))
    y = rng.standard_normal((3, H, W))
    k = synth.gaussian_kernel(9, 1.6).astype(np.float64)
    x = operators.blur_prox(v, y, k, tau)
    res = x + tau * operators.blur_grad(x, y, k) - v
    assert np.linalg.norm(res) <= 1e-12 * np.linalg.norm(v)
    m = synth.bernoulli_mask(rng, H, W).astype(np.float64)[None]
    x = operators.inpaint_prox(v, y * m, m, tau)
    res = x + tau * operators.inpaint_grad(x, y * m, m) - v
    assert np.linalg.norm(res) <= 1e-12 * np.linalg.norm(v)
    # missing pixels keep the iterate
    assert np.array_equal(x[np.broadcast_to(m == 0, x.shape)], v[np.broadcast_to(m == 0, v.shape)])


# ----------------------------------------------------------------------------- P8
def test_P8_merit_decrease_beta0():
    """P8: beta = 0, gradient variant, tau < 1/L: F = f + lam g (Eq. 1) obeys the descent
    lemma F(x+) <= F(x) - tau(1 - tau L/2)||grad F||^2 at every step."""
    net, _ = _tiny(scale=0.5)
    rng = np.random.default_rng(11)
    x = rng.uniform(0, 1, (1, 16, 16))
    k = synth.gaussian_kernel(9, 1.6).astype(np.float64)
    fid = operators.Fidelity("blur", operators.blur_A(x, k) + 0.01 * rng.standard_normal(x.shape), kernel=k)
    lam = 0.5
    # L_g by power iteration on finite-difference Hessian-vector products, then a 2x margin.
    v = rng.standard_normal(x.shape)
    for _ in range(30):
        hv = (net.grad_g(x + 1e-5 * v) - net.grad_g(x - 1e-5 * v)) / 2e-5
        Lg = np.linalg.norm(hv) / np.linalg.norm(v)
        v = hv
    L = 1.0 + lam * 2.0 * Lg
    tau = 0.9 / L

    def F(u):
        return fid.value(u) + lam * net.g(u)
    xk = fid.y.copy()
    for _ in range(30):
        gF = fid.grad(xk) + lam * net.grad_g(xk)
        xn = xk - tau * gF
        assert F(xn) <= F(xk) - tau * (1 - tau * L / 2) * float(np.sum(gF * gF)) + 1e-12
        xk = xn


# ----------------------------------------------------------------------------- P9
def test_P9_spec_worked_examples():
    gold = json.load(open(GOLD))
    m = gold["momentum"]
    beta = 1.0 - m["alpha"]
    assert m["x_curr"] + beta * (m["x_curr"] - m["x_prev"]) == pytest.approx(m["z"], abs=1e-15)

    # the oracle's own extrapolation (Eq. 4) on the same example: with tau = 0 the
    # operator returns z^k exactly.
    net0, _ = _tiny(C=1, w=4, scale=0.0, skip=False)
    fid0 = operators.Fidelity("blur", np.zeros((1, 1, 1)), kernel=np.ones((1, 1)))
    z = solver.ideq_step(np.full((1, 1, 1), m["x_curr"]), np.full((1, 1, 1), m["x_prev"]),
                         net0, fid0, 0.05, 0.0, beta, "grad")
    assert z.item() == pytest.approx(m["z"], abs=1e-15)
    # residual definition (Q3): ||x^{k+1} - x^k|| / ||x^k||
    assert solver.residual(np.array([3.0, 4.0]) * 2, np.array([3.0, 4.0])) == 1.0
    assert solver.residual(np.ones(2), np.zeros(2)) == float("inf")

    r = gold["red_step_scalar"]
    z = np.array([[[r["z"]]]])
    # tikhonov g = x^2/2 via the zero-output net without skip; f = (x-y)^2/2 via a 1x1 identity blur
    net, _ = _tiny(C=1, w=4, scale=0.0, skip=False)
    fid = operators.Fidelity("blur", np.array([[[r["y"]]]]), kernel=np.ones((1, 1)))
    xn = solver.ideq_step(z, z, net, fid, r["lambda"], r["tau"], 0.0, "grad")
    assert xn.item() == r["x_next"]

    p = gold["inpaint_prox_all_ones"]
    y = np.array(p["y"])[None, None]
    v = np.array(p["v"])[None, None]
    out = operators.inpaint_prox(v, y, np.ones((1, 1, 3)), p["tau"])
    assert np.allclose(out.ravel(), p["prox"], atol=1e-15)

    t = gold["tikhonov_fixed_point"]
    yy = np.random.default_rng(12).uniform(0, 1, (1, 8, 8))
    fid = operators.Fidelity("blur", yy, kernel=np.ones((1, 1)))
    out = solver.solve(net, [fid], yy[None], t["lambda"], 0.9, 0.5, 500, 0.0, "grad")
    assert np.abs(out["x"][0] - yy / (1 + t["lambda"])).max() <= t["tol"]


# ----------------------------------------------------------------------------- P10
def test_P10_phase_gradient():
    """P10: FD check of the phase-retrieval gradient (incl. the factor 2) and
    grad f(x_true; y_clean) = 0."""
    rng = np.random.default_rng(13)
    H = W = 16
    D = synth.phase_masks(rng, 4, H, W).astype(np.float64)
    Dc = D[..., 0] + 1j * D[..., 1]
    x = rng.uniform(0, 1, (1, H, W))
    y_clean = np.abs(np.fft.fft2(Dc * x[0][None], norm="ortho")) ** 2
    assert np.abs(operators.phase_grad(x, y_clean, Dc)).max() <= 1e-12
    y = y_clean + 0.05 * rng.standard_normal(y_clean.shape)
    xq = x + 0.1 * rng.standard_normal(x.shape)
    g = operators.phase_grad(xq, y, Dc)
    h = 1e-5
    for _ in range(10):
        d = rng.standard_normal(x.shape)
        d /= np.linalg.norm(d)
        fd = (operators.phase_f(xq + h * d, y, Dc) - operators.phase_f(xq - h * d, y, Dc)) / (2 * h)
        an = float(np.sum(g * d))
        assert abs(fd - an) <= 1e-6 * (1 + abs(an))


def test_P10_blur_inpaint_grad_fd():
    rng = np.random.default_rng(14)
    x = rng.uniform(0, 1, (3, 12, 12))
    y = rng.uniform(0, 1, (3, 12, 12))
    k = synth.motion_kernel(rng, 15)
    m = synth.bernoulli_mask(rng, 12, 12)
    for fid in (operators.Fidelity("blur", y, kernel=k), operators.Fidelity("inpaint", y * m[None], mask=m)):
        g = fid.grad(x)
        for _ in range(5):
            d = rng.standard_normal(x.shape)
            d /= np.linalg.norm(d)
            fd = (fid.value(x + 1e-5 * d) - fid.value(x - 1e-5 * d)) / 2e-5
            an = float(np.sum(g * d))
            assert abs(fd - an) <= 1e-6 * (1 + abs(an))


# ----------------------------------------------------------------------------- P11
def test_P11_batch_independence():
    """P11: the per-image rule makes a batched solve equal to per-image solves, bit for bit."""
    from paper_2605_19705_b200 import configs
    cfg = configs.get("C3", batch=3, H=16, W=16, widths=(8, 8, 8, 8), max_iter=12, tol=1e-3)
    prob = synth.make_problem(cfg)
    net = solver.make_net(cfg, prob["weights"])
    fids = solver.make_fidelities(cfg, prob)
    full = solver.solve(net, fids, prob["x0"], cfg["lam"], cfg["tau"], cfg["beta"], 12, 1e-3, "prox")
    for b in range(3):
        one = solver.solve(net, [fids[b]], prob["x0"][b:b + 1], cfg["lam"], cfg["tau"], cfg["beta"], 12, 1e-3, "prox")
        assert np.array_equal(one["x"][0], full["x"][b])
        assert one["iters"][0] == full["iters"][b]


def test_stop_rules_and_divergence():
    """Reading Q17 / Q22: per-image freeze, global-max rule, non-finite freeze at the last finite iterate."""
    net, _ = _tiny(scale=0.0, skip=False)                       # g = 1/2||x||^2
    rng = np.random.default_rng(15)
    ys = rng.uniform(0.5, 1, (2, 1, 4, 4))
    fids = [operators.Fidelity("blur", ys[b], kernel=np.ones((1, 1))) for b in range(2)]
    out = solver.solve(net, fids, ys, 0.05, 0.9, 0.0, 200, 1e-6, "grad", 1, "per_image")
    assert (out["status"] == solver.CONVERGED).all() and (out["residual"] <= 1e-6).all()
    out_g = solver.solve(net, fids, ys, 0.05, 0.9, 0.0, 200, 1e-6, "grad", 10, "global_max")
    assert (out_g["iters"] % 10 == 0).all() and len(set(out_g["iters"])) == 1
    # divergence: a huge step makes the iterate overflow
    bad = solver.solve(net, fids, ys, 1e300, 1e10, 0.0, 10, 0.0, "grad")
    assert (bad["status"] == solver.DIVERGED).all()
    assert np.isfinite(bad["x"]).all()
