"""CPU pins of the oracle's adaptive restart (Eq. 5) and averaging (Alg. 1/2 steps 12-13),
SURVEY §8(f) NEXT-1. Each pin is fixed by the paper's definitions or a closed form, not by the
oracle itself:
  - restart arithmetic: SPEC's worked example k = 3, increments {1, 2, 2}, B = 5 -> 27 > 25;
  - B = inf is the no-restart loop; B = 0 with either semantics removes all inertia, so the
    iterates equal a separately written RED loop (Eq. 3) bit for bit;
  - Alg. 1 vs Alg. 2 state transitions: after the first restart Alg. 2 (x^{k-1} <- x^k only, the
    counter and sum keep growing) restarts at every later iteration;
  - averaging on x^{k+1} = x^k - tau (x^k - y) (beta = 0, lambda = 0, all-ones inpainting mask):
    x^k = y + (1-tau)^k (x^0 - y), increments decrease, K0 = K - 2 and
    x_hat = y + (x^0 - y) (1 - (1-tau)^{K-1}) / (tau (K-1)) (geometric series);
  - empty window (K <= 4) -> x^K; constant iterates -> x_hat = that constant, K0 = floor(K/2)+1.
"""
import numpy as np
import pytest

from oracle import solver as osolver
from oracle.operators import Fidelity
from paper_2605_19705_b200 import configs, synth


def test_restart_check_worked_example():
    # SPEC: k = 3, increments of norms {1, 2, 2}, B = 5 -> 3 * 9 = 27 > 25
    assert osolver.restart_check(3, 1.0 + 4.0 + 4.0, 5.0)
    assert not osolver.restart_check(3, 1.0 + 4.0 + 4.0, 5.2)      # 27 < 27.04
    assert not osolver.restart_check(10, 1e6, float("inf"))
    assert osolver.restart_check(1, 1e-30, 0.0)


def _c1(**kw):
    cfg = configs.get("C1", **kw)
    prob = synth.make_problem(cfg)
    return cfg, prob


@pytest.mark.parametrize("mode", [1, 2])
def test_restart_never_triggers_with_infinite_B(mode):
    cfg, prob = _c1()
    a = osolver.solve_config(cfg, prob, max_iter=25, tol=0.0)
    b = osolver.solve_config(cfg, prob, max_iter=25, tol=0.0, restart=mode, restart_B=float("inf"))
    assert np.array_equal(a["x"], b["x"]) and b["restarts"][0] == 0


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("name", ["C1", "C3"])
def test_restart_every_step_is_red(mode, name):
    """B = 0: every accepted step with a nonzero increment restarts, so z^k = x^k always and the
    inertial loop IS the RED / RED-P loop (Eq. 3) -- bitwise, over 30 iterations."""
    kw = dict(batch=1, H=16, W=24) if name == "C3" else {}
    cfg = configs.get(name, **kw)
    prob = synth.make_problem(cfg)
    K = 30
    out = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, restart=mode, restart_B=0.0)
    net = osolver.make_net(cfg, prob["weights"])
    fid = osolver.make_fidelities(cfg, prob)[0]
    x = prob["x0"][0].astype(np.float64)
    for _ in range(K):                                   # plain RED / RED-P, written out
        gg = net.grad_g(x)
        if cfg["step"] == "grad":
            x = x - cfg["tau"] * (fid.grad(x) + cfg["lam"] * gg)
        else:
            x = fid.prox(x - cfg["tau"] * cfg["lam"] * gg, cfg["tau"])
    assert np.array_equal(out["x"][0], x)
    assert out["restarts"][0] == K


def test_alg1_vs_alg2_restart_state():
    """Alg. 2 keeps k and the sum after a restart, so once Eq. 5 holds it holds at every later
    iteration; Alg. 1 resets both and restarts less often."""
    cfg, prob = _c1()
    K = 40
    ref = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0)
    # B between the first-iteration increment and the accumulated criterion: a few restarts
    x0 = prob["x0"][0].astype(np.float64)
    B = 0.5 * np.linalg.norm(ref["x"][0] - x0)
    a1 = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, restart=1, restart_B=B)
    a2 = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, restart=2, restart_B=B)
    assert a1["restarts"][0] >= 1
    assert a2["restarts"][0] >= a1["restarts"][0]
    # Alg. 2: restarts are a contiguous tail of the iterations
    net = osolver.make_net(cfg, prob["weights"])
    fid = osolver.make_fidelities(cfg, prob)[0]
    xc = xp = x0
    ks, S, first = 0, 0.0, None
    for k in range(K):
        xn = osolver.ideq_step(xc, xp, net, fid, cfg["lam"], cfg["tau"], cfg["beta"], cfg["step"])
        ks += 1
        S += float(np.sum((xn - xc) ** 2))
        if ks * S > B * B:
            first = k if first is None else first
            xp = xc = xn
        else:
            xp, xc = xc, xn
    assert first is not None and a2["restarts"][0] == K - first
    assert np.array_equal(a2["x"][0], xc)


def _contraction_problem(H=8, W=8, seed=0):
    rng = np.random.default_rng(seed)
    y = rng.uniform(0, 1, (1, H, W))
    x0 = rng.uniform(0, 1, (1, H, W))
    fid = Fidelity("inpaint", y, mask=np.ones((H, W), dtype=np.uint8))   # grad f = x - y

    class ZeroNet:                                                       # lambda = 0 anyway
        def grad_g(self, z):
            return np.zeros_like(z)
    return y, x0, fid, ZeroNet()


@pytest.mark.parametrize("K,tau", [(10, 0.3), (17, 0.45), (30, 0.1)])
def test_averaging_geometric_closed_form(K, tau):
    y, x0, fid, net = _contraction_problem()
    out = osolver.solve(net, [fid], x0[None], 0.0, tau, 0.0, K, 0.0, "grad", averaging=True)
    assert out["k0"][0] == K - 2
    want = y + (x0 - y) * (1.0 - (1.0 - tau) ** (K - 1)) / (tau * (K - 1))
    assert np.allclose(out["x"][0], want, rtol=0, atol=1e-13)


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_averaging_empty_window_returns_last_iterate(K):
    y, x0, fid, net = _contraction_problem()
    a = osolver.solve(net, [fid], x0[None], 0.0, 0.3, 0.0, K, 0.0, "grad", averaging=True)
    b = osolver.solve(net, [fid], x0[None], 0.0, 0.3, 0.0, K, 0.0, "grad")
    assert a["k0"][0] == -1 and np.array_equal(a["x"], b["x"])


def test_averaging_constant_iterates_and_tie_break():
    y, _, fid, net = _contraction_problem()
    K = 12
    # tol < 0: r = 0 exactly must not count as converged (tol = 0 would stop at r <= 0)
    out = osolver.solve(net, [fid], y[None], 0.0, 0.3, 0.5, K, -1.0, "grad", averaging=True)
    assert out["k0"][0] == K // 2 + 1                                    # all increments 0: lowest k
    assert np.allclose(out["x"][0], y, rtol=0, atol=1e-15)             # mean of equal planes


def test_averaging_requires_fixed_count():
    y, x0, fid, net = _contraction_problem()
    with pytest.raises(ValueError):
        osolver.solve(net, [fid], x0[None], 0.0, 0.3, 0.0, 10, 1e-4, "grad", averaging=True)
