"""GPU-vs-oracle parity of NEXT-1: adaptive restart (Eq. 5) with the
Alg. 1 and Alg. 2 semantics, and the averaging steps 12-13, through
the C ABI (ideq_params.restart / restart_B / averaging)."""
import numpy as np
import pytest

from oracle import solver as osolver
from paper_2605_19705_b200 import configs, synth
from tests.gpu_util import psnr, rel_l2, torch_cuda

pytestmark = pytest.mark.gpu


def _dev(torch, a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _setup(name, precision, **kw):
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    base = dict(C1=dict(), C3=dict(batch=2, H=48, W=40), C5=dict(batch=2, H=64, W=128))[name]
    base.update(kw)
    cfg = configs.get(name, **base)
    prob = synth.make_problem(cfg)
    s = ideq.Solver(cfg, prob["weights"], precision=precision, max_batch=cfg["batch"])
    s.set_operator(prob)
    return torch, cfg, prob, s


def _run(torch, s, prob, **pk):
    xd = _dev(torch, prob["x0"])
    st, code, _ = s.solve(_dev(torch, prob["y"]), xd, s.params(**pk))
    return st, code, xd.cpu().numpy()


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("name", ["C1", "C3", "C5"])
def test_restart_matches_oracle_fp32(name, mode):
    torch, cfg, prob, s = _setup(name, "fp32", init_scale=0.3)
    K = 24
    lam = configs.STRESS[name]["lam"]
    ref = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, lam=lam)
    x0 = prob["x0"][0].astype(np.float64)
    B = 0.5 * float(np.linalg.norm(ref["x"][0] - x0))
    orc = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, lam=lam, restart=mode, restart_B=B)
    st, code, x = _run(torch, s, prob, lam=lam, max_iter=K, tol=0.0, restart=mode, restart_B=B)
    assert (orc["restarts"] >= 1).all()
    assert np.array_equal(st["restarts"], orc["restarts"])
    for b in range(x.shape[0]):
        assert rel_l2(x[b], orc["x"][b]) <= 1e-4
        assert abs(st["residual"][b] - orc["residual"][b]) <= 1e-6


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_restart_every_step_equals_beta_zero(precision):
    """B = 0: every step restarts, z^{k+1} := x^{k+1}, i.e. the beta = 0 (RED-P) iteration -- the
    GPU's own beta = 0 run, bit for bit."""
    torch, cfg, prob, s = _setup("C3", precision)
    st_a, _, xa = _run(torch, s, prob, max_iter=12, tol=0.0, restart=1, restart_B=0.0)
    st_b, _, xb = _run(torch, s, prob, max_iter=12, tol=0.0, beta=0.0)
    assert np.array_equal(xa, xb)
    assert (st_a["restarts"] == 12).all()


@pytest.mark.parametrize("name,K", [("C1", 30), ("C3", 14), ("C5", 11)])
def test_averaging_matches_oracle_fp32(name, K):
    torch, cfg, prob, s = _setup(name, "fp32")
    orc = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, averaging=True)
    st, code, x = _run(torch, s, prob, max_iter=K, tol=0.0, averaging=True)
    assert np.array_equal(st["k0"], orc["k0"]) and (orc["k0"] > K // 2).all()
    for b in range(x.shape[0]):
        assert rel_l2(x[b], orc["x"][b]) <= 1e-4


def test_averaging_with_restart_bf16_psnr():
    torch, cfg, prob, s = _setup("C3", "bf16")
    K = 16
    orc = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, restart=1, restart_B=0.05, averaging=True)
    st, code, x = _run(torch, s, prob, max_iter=K, tol=0.0, restart=1, restart_B=0.05, averaging=True)
    for b in range(x.shape[0]):
        d = abs(psnr(x[b], prob["x_true"][b]) - psnr(orc["x"][b], prob["x_true"][b]))
        assert d <= 0.05, d


def test_averaging_needs_fixed_count_and_window():
    torch, cfg, prob, s = _setup("C3", "fp32")
    from paper_2605_19705_b200 import ideq
    with pytest.raises(ideq.IdeqError) as ei:
        _run(torch, s, prob, max_iter=10, tol=1e-4, averaging=True)
    assert ei.value.code == ideq.E_INVALID
    # K = 4: empty window -> x-hat = x^K, K0 = -1
    st, _, xa = _run(torch, s, prob, max_iter=4, tol=0.0, averaging=True)
    _, _, xb = _run(torch, s, prob, max_iter=4, tol=0.0)
    assert (st["k0"] == -1).all() and np.array_equal(xa, xb)


def test_averaging_two_solves_different_max_iter_one_solver():
    """The CUDA graph of an iteration bakes in the finalize arguments, among them the averaging
    window K = max_iter: a second solve on the SAME context with another max_iter must not
    reuse the first solve's graph. Both solves are checked against the oracle (K0 and x-hat)."""
    torch, cfg, prob, s = _setup("C3", "fp32")
    for K in (5, 14, 9):
        orc = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, averaging=True)
        st, code, x = _run(torch, s, prob, max_iter=K, tol=0.0, averaging=True)
        assert np.array_equal(st["k0"], orc["k0"]), (K, st["k0"], orc["k0"])
        for b in range(x.shape[0]):
            assert rel_l2(x[b], orc["x"][b]) <= 1e-4, K
