"""GPU-vs-oracle parity of NEXT-4: the JFB training gradient at x_hat
 through the C ABI `ideq_jfb_grad`, against oracle/jfb.py (fp64,
itself pinned to torch double-backward and to finite differences in test_oracle_jfb.py).

Tolerance (fp32 path vs fp64 oracle): the weight gradient is a sum over every pixel of products of
O(1) fp32 terms, so its relative L2 error is ~sqrt(#terms) * 2^-24 ~ 1e-5..1e-4 at these sizes;
the test takes 1e-3 on the whole vector and per weight tensor. Scalars (sums reduced in fp64 from
fp32 terms): 1e-4 relative.
"""
import numpy as np
import pytest

from oracle import jfb
from oracle import solver as osolver
from paper_2605_19705_b200 import configs, synth
from tests.gpu_util import rel_l2, torch_cuda

pytestmark = pytest.mark.gpu


def _dev(torch, a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


CASES = [("C1", "grad", dict(batch=2)),
         ("C3", "grad", dict(batch=2, H=32, W=32, widths=(32, 32, 64, 64))),
         ("C3", "prox", dict(batch=2, H=32, W=48, widths=(32, 32, 64, 64))),
         ("C3", "prox", dict(batch=1))]          # full C3 size: 256^2 RGB, U-Net-32 (oracle ~5 s)


@pytest.mark.parametrize("name,step,kw", CASES)
def test_jfb_grad_parity(name, step, kw):
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    cfg = configs.get(name, init_scale=0.3, step=step, **kw)
    prob = synth.make_problem(cfg)
    s = ideq.Solver(cfg, prob["weights"], precision="fp32", max_batch=cfg["batch"])
    s.set_operator(prob)
    xs = prob["x_true"].astype(np.float32)
    x_hat = (0.9 * xs + 0.05 + 0.02 * np.random.default_rng(5).standard_normal(xs.shape)).astype(np.float32)
    lam, tau = 0.7, 0.6
    loss, dth, dlam, dtau, dbeta = s.jfb_grad(_dev(torch, prob["y"]), _dev(torch, x_hat), _dev(torch, xs),
                                              s.params(lam=lam, tau=tau))
    again = s.jfb_grad(_dev(torch, prob["y"]), _dev(torch, x_hat), _dev(torch, xs), s.params(lam=lam, tau=tau))
    assert np.array_equal(again[1], dth) and again[0] == loss    # pooled scratch reused: deterministic
    net = osolver.make_net(cfg, prob["weights"])
    fids = osolver.make_fidelities(cfg, prob)
    want = [jfb.jfb_grads(net, fids[b], x_hat[b].astype(np.float64), xs[b].astype(np.float64), lam, tau, step)
            for b in range(cfg["batch"])]
    w_loss = sum(w[0] for w in want)
    w_dth = sum(w[1] for w in want)
    w_dlam = sum(w[2] for w in want)
    w_dtau = sum(w[3] for w in want)
    assert dbeta == 0.0
    assert abs(loss - w_loss) <= 1e-4 * abs(w_loss)
    assert abs(dlam - w_dlam) <= 1e-4 * (abs(w_dlam) + 1e-3 * w_loss)
    assert abs(dtau - w_dtau) <= 1e-4 * (abs(w_dtau) + 1e-3 * w_loss)
    assert np.all(np.isfinite(dth))
    assert rel_l2(dth, w_dth) <= 1e-3
    off = 0
    for k, w in net.W.items():          # every tensor, so a mis-permuted layer cannot hide
        sl = slice(off, off + w.size)
        off += w.size
        assert rel_l2(dth[sl], w_dth[sl]) <= 1e-3, k
    assert off == dth.size


def test_jfb_grad_rejects_bf16_and_non_inpaint_prox():
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    cfg = configs.get("C3", batch=1, H=32, W=32)
    prob = synth.make_problem(cfg)
    s = ideq.Solver(cfg, prob["weights"], precision="bf16", max_batch=1)
    s.set_operator(prob)
    x = _dev(torch, prob["x_true"])
    with pytest.raises(ideq.IdeqError, match="UNSUPPORTED"):
        s.jfb_grad(_dev(torch, prob["y"]), x, x, s.params())
    cfg = configs.get("C5", batch=1, H=32, W=32, step="prox", widths=(32, 32, 64, 64))
    prob = synth.make_problem(cfg)
    s = ideq.Solver(cfg, prob["weights"], precision="fp32", max_batch=1)
    s.set_operator(prob)
    x = _dev(torch, prob["x_true"])
    with pytest.raises(ideq.IdeqError, match="UNSUPPORTED"):
        s.jfb_grad(_dev(torch, prob["y"]), x, x, s.params())
