"""Fused level-0 residual blocks (csrc/rbf.cu): the block's two 3x3 convolutions in one launch,
streamed down full image rows (the network of Eq. 2, and its
input VJP). Checked (1) per block against the oracle's layer definitions composed (oracle/nets.py),
element by element, (2) inside the solver against the same network run as two launches per
block (ideq_debug_set_fusion), and (3) as the solver's default path by every bf16 U-Net test
(trajectories, live list, full size)."""
import numpy as np
import pytest

from oracle import nets
from paper_2605_19705_b200 import configs, synth
from tests.gpu_util import bf16_round, from_nhwc_dev, nhwc_dev, rel_l2, torch_cuda

pytestmark = pytest.mark.gpu


def _elementwise(got, ref):
    assert np.isfinite(got).all()
    bound = 2.0 ** -8 * np.abs(ref).max()
    err = np.abs(got - ref)
    assert err.max() <= bound, (float(err.max()), float(bound), np.unravel_index(err.argmax(), err.shape))


@pytest.mark.parametrize("W,H,N", [(128, 13, 2), (256, 7, 3), (256, 1, 2), (128, 40, 1), (128, 5, 70), (256, 3, 150)])
def test_fused_block_forward(W, H, N):
    """a = sp(A x) (saved), out = x + B a: H ragged against the per-CTA row runs, a single row, runs
    crossing image boundaries."""
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    rng = np.random.default_rng(W + 7 * H + N)
    wA = (rng.standard_normal((32, 32, 3, 3)) * np.sqrt(2.0 / 288)).astype(np.float32)
    wB = (rng.standard_normal((32, 32, 3, 3)) * np.sqrt(2.0 / 288)).astype(np.float32)
    x = rng.standard_normal((N, 32, H, W))
    xr, ar, br = bf16_round(x), bf16_round(wA), bf16_round(wB)
    a_ref = np.stack([nets.softplus(nets.conv3x3(xr[n], ar)) for n in range(N)])
    a_rb = bf16_round(a_ref)  # the kernel keeps a in bf16 (as the unfused layer stores it)
    out_ref = np.stack([xr[n] + nets.conv3x3(a_rb[n], br) for n in range(N)])
    xd = nhwc_dev(x, "bf16")
    out = torch.zeros_like(xd)
    act = torch.zeros_like(xd)
    ideq.debug_rb(False, wA, wB, N, H, W, xd, out, act)
    _elementwise(from_nhwc_dev(act), a_ref)
    _elementwise(from_nhwc_dev(out), out_ref)
    assert rel_l2(from_nhwc_dev(out), out_ref) <= 8e-3


@pytest.mark.parametrize("W,H,N", [(128, 13, 2), (256, 9, 2), (128, 5, 70), (256, 3, 150)])
def test_fused_block_vjp(W, H, N):
    """q = (B^T g) . sp'(a) with sp'(a) = 1 - exp(-a) from the saved activation, out = g + A^T q."""
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    rng = np.random.default_rng(100 + W + H)
    wA = (rng.standard_normal((32, 32, 3, 3)) * np.sqrt(2.0 / 288)).astype(np.float32)
    wB = (rng.standard_normal((32, 32, 3, 3)) * np.sqrt(2.0 / 288)).astype(np.float32)
    g = rng.standard_normal((N, 32, H, W))
    a = rng.uniform(0.05, 2.0, (N, 32, H, W))
    gr, arr, wa, wb = bf16_round(g), bf16_round(a), bf16_round(wA), bf16_round(wB)
    q = np.stack([nets.conv3x3_T(gr[n], wb) * (-np.expm1(-arr[n])) for n in range(N)])
    out_ref = np.stack([gr[n] + nets.conv3x3_T(bf16_round(q)[n], wa) for n in range(N)])
    gd = nhwc_dev(g, "bf16")
    ad = nhwc_dev(a, "bf16")
    out = torch.zeros_like(gd)
    ideq.debug_rb(True, wA, wB, N, H, W, gd, out, ad)
    got = from_nhwc_dev(out)
    _elementwise(got, out_ref)
    assert rel_l2(got, out_ref) <= 8e-3


@pytest.mark.parametrize("name,kw", [("C3", dict(batch=3, H=24, W=128)), ("C3", dict(batch=2, H=16, W=256)),
                                     ("C2", dict(batch=2, H=128, W=128))])
def test_fused_blocks_match_two_launches_in_solver(name, kw):
    """The solver's bf16 network with fused level-0 blocks vs the same network run as two launches
    per block: grad g and a 4-iteration trajectory (stress init so the network matters)."""
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    cfg = configs.get(name, init_scale=configs.STRESS[name]["init_scale"], **kw)
    prob = synth.make_problem(cfg)
    res = []
    for fuse in (True, False):
        s = ideq.Solver(cfg, prob["weights"], precision="bf16", max_batch=cfg["batch"])
        s.set_fusion(fuse)
        s.set_operator(prob)
        z = torch.tensor(prob["x_true"].astype(np.float32)).cuda()
        g = torch.zeros_like(z)
        s.grad_g(z, g)
        x = torch.tensor(prob["x0"].astype(np.float32)).cuda()
        s.solve(torch.tensor(prob["y"].astype(np.float32)).cuda(), x,
                s.params(lam=configs.STRESS[name]["lam"], max_iter=4, tol=0.0))
        res.append((g.cpu().numpy(), x.cpu().numpy()))
        s.close()
    # Not bit-identical: the fused kernel sums a 3x3 convolution as three row-partial sums (taps of
    # one kernel row in one N = 96 GEMM, shifted and added in the epilogue), a different fp32 order
    # than the 9-tap accumulation of the two-launch path, so bf16-rounded intermediates flip by one
    # ulp on near-ties and the stress-init network amplifies that. Bound: a third of the bf16
    # network's bound against the oracle (3e-2, test_gpu_parity.test_grad_g_component).
    assert rel_l2(res[0][0], res[1][0]) <= 1e-2, rel_l2(res[0][0], res[1][0])
    assert rel_l2(res[0][1], res[1][1]) <= 1e-2, rel_l2(res[0][1], res[1][1])
