"""GPU-vs-oracle parity of NEXT-2: the Rician fidelity of App. D.3.3
 fused into the gradient step (Alg. 1), through the C ABI."""
import numpy as np
import pytest

from oracle import solver as osolver
from paper_2605_19705_b200 import configs, synth
from tests.gpu_util import psnr, rel_l2, torch_cuda

pytestmark = pytest.mark.gpu


def _dev(torch, a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _setup(precision, **kw):
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    base = dict(batch=3, H=48, W=40)
    base.update(kw)
    cfg = configs.get("R1", **base)
    prob = synth.make_problem(cfg)
    s = ideq.Solver(cfg, prob["weights"], precision=precision, max_batch=cfg["batch"])
    s.set_operator(prob)
    return torch, cfg, prob, s


def test_rician_gradient_component():
    torch, cfg, prob, s = _setup("fp32")
    fids = osolver.make_fidelities(cfg, prob)
    x = (0.9 * prob["x_true"] + 0.05).astype(np.float32)
    out = torch.zeros_like(_dev(torch, x))
    s.fidelity_grad(_dev(torch, prob["y"]), _dev(torch, x), out)
    for b in range(x.shape[0]):
        assert rel_l2(out[b].cpu().numpy(), fids[b].grad(x[b].astype(np.float64))) <= 1e-5


@pytest.mark.parametrize("stress", [False, True])
def test_rician_trajectory_fp32(stress):
    kw = dict(init_scale=configs.STRESS["R1"]["init_scale"]) if stress else {}
    lam = configs.STRESS["R1"]["lam"] if stress else None
    torch, cfg, prob, s = _setup("fp32", **kw)
    K = 12
    xd = _dev(torch, prob["x0"])
    st, code, _ = s.solve(_dev(torch, prob["y"]), xd, s.params(lam=lam, max_iter=K, tol=0.0))
    orc = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, lam=lam)
    x = xd.cpu().numpy()
    for b in range(x.shape[0]):
        assert rel_l2(x[b], orc["x"][b]) <= 1e-4
        assert abs(st["residual"][b] - orc["residual"][b]) <= 1e-6


def test_rician_bf16_psnr_and_no_prox():
    torch, cfg, prob, s = _setup("bf16")
    from paper_2605_19705_b200 import ideq
    K = 20
    xd = _dev(torch, prob["x0"])
    s.solve(_dev(torch, prob["y"]), xd, s.params(max_iter=K, tol=0.0))
    orc = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0)
    x = xd.cpu().numpy()
    for b in range(x.shape[0]):
        d = abs(psnr(x[b], prob["x_true"][b]) - psnr(orc["x"][b], prob["x_true"][b]))
        assert d <= 0.05, d
    with pytest.raises(ideq.IdeqError) as ei:          # no closed-form prox
        s.set_operator(prob, step="prox")
    assert ei.value.code == ideq.E_UNSUPPORTED
