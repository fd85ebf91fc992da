"""GPU-vs-oracle parity of NEXT-3: the compressed-sensing MRI fidelity of App.
D.3.1 -- k-space gradient and closed-form prox (reading Q18) on the half-spectrum
FFT passes -- in both the gradient (Alg. 1) and proximal (Alg. 2) variants, through the C ABI."""
import numpy as np
import pytest

from oracle import solver as osolver
from paper_2605_19705_b200 import configs, synth
from tests.gpu_util import psnr, rel_l2, torch_cuda

pytestmark = pytest.mark.gpu


def _dev(torch, a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _setup(precision, step="prox", **kw):
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    base = dict(batch=3, H=64, W=32, step=step)
    base.update(kw)
    cfg = configs.get("M1", **base)
    prob = synth.make_problem(cfg)
    s = ideq.Solver(cfg, prob["weights"], precision=precision, max_batch=cfg["batch"])
    s.set_operator(prob)
    return torch, cfg, prob, s


def test_mri_components():
    torch, cfg, prob, s = _setup("fp32")
    fids = osolver.make_fidelities(cfg, prob)
    # away from the truth, where grad f (a difference of two nearly equal k-space terms) is at the
    # noise level and fp32 cancellation dominates its relative error
    x = (0.9 * prob["x_true"] + 0.05).astype(np.float32)
    out = torch.zeros_like(_dev(torch, x))
    s.fidelity_grad(_dev(torch, prob["y"]), _dev(torch, x), out)
    for b in range(x.shape[0]):
        assert rel_l2(out[b].cpu().numpy(), fids[b].grad(x[b].astype(np.float64))) <= 1e-5
    s.fidelity_prox(_dev(torch, prob["y"]), _dev(torch, x), 0.7, out)
    for b in range(x.shape[0]):
        assert rel_l2(out[b].cpu().numpy(), fids[b].prox(x[b].astype(np.float64), 0.7)) <= 2e-6


@pytest.mark.parametrize("step", ["prox", "grad"])
@pytest.mark.parametrize("stress", [False, True])
def test_mri_trajectory_fp32(step, stress):
    kw = dict(init_scale=configs.STRESS["M1"]["init_scale"]) if stress else {}
    lam = configs.STRESS["M1"]["lam"] if stress else None
    torch, cfg, prob, s = _setup("fp32", step=step, **kw)
    K = 10
    xd = _dev(torch, prob["x0"])
    st, code, _ = s.solve(_dev(torch, prob["y"]), xd, s.params(lam=lam, max_iter=K, tol=0.0))
    orc = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, lam=lam)
    x = xd.cpu().numpy()
    for b in range(x.shape[0]):
        assert rel_l2(x[b], orc["x"][b]) <= 1e-4
        assert abs(st["residual"][b] - orc["residual"][b]) <= 1e-6


def test_mri_bf16_psnr_and_mask_check():
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
    bad = dict(prob)
    km = prob["kmask"].copy()
    km[1, 3] = 1 - km[1, 3]                               # breaks M[-ky][-kx] == M[ky][kx]
    bad["kmask"] = km
    with pytest.raises(ideq.IdeqError) as ei:
        s.set_operator(bad)
    assert ei.value.code == ideq.E_INVALID
