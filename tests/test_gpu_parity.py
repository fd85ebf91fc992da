"""GPU-vs-oracle parity through the C ABI.

fp32 mode: component grad g within 1e-5 relative; iterates after K steps within 1e-4
relative L2 and final residual within 1e-6 absolute (BASELINE north_star).
bf16 mode: PSNR of the reconstruction within 0.05 dB of the oracle's (north_star);
component grad g documented at <= 3e-2 relative.
Sizes are reduced versions of C1..C4 that span several tiles and ragged tails."""
import numpy as np
import pytest

from oracle import solver as osolver
from paper_2605_19705_b200 import configs, synth
from tests.gpu_util import psnr, rel_l2, torch_cuda

pytestmark = pytest.mark.gpu

# step size of the reduced phase-retrieval case (tools/freeze_tau_pr.py rule on the mini problem)
TAU_PR_MINI = 0.5 / 21


def _mini(name, **kw):
    base = dict(C1=dict(), C2=dict(batch=2, H=48, W=40), C3=dict(batch=2, H=48, W=40),
                C4=dict(batch=2, H=64, W=32, tau=TAU_PR_MINI), C5=dict(batch=2, H=64, W=128))[name]
    base.update(kw)
    return configs.get(name, **base)


def _solver(cfg, prob, precision):
    from paper_2605_19705_b200 import ideq
    s = ideq.Solver(cfg, prob["weights"], precision=precision, max_batch=len(prob["images"]))
    s.set_operator(prob)
    return s


def _dev(torch, a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


@pytest.mark.parametrize("name,precision,tol", [("C1", "fp32", 1e-5), ("C3", "fp32", 1e-5), ("C3", "bf16", 3e-2),
                                                ("C2", "bf16", 3e-2)])
@pytest.mark.parametrize("scale", [0.1, 0.3])
def test_grad_g_component(name, precision, tol, scale):
    """grad g(z) = (I - J_N)^T (z - N(z)) (Eq. 2) on the same z; scale 0.3 (the stress
    init) exercises the nonlinearity harder than the BASELINE x0.1 init."""
    torch = torch_cuda()
    cfg = _mini(name, init_scale=scale)
    prob = synth.make_problem(cfg)
    s = _solver(cfg, prob, precision)
    z = prob["x_true"].astype(np.float32)
    zd = _dev(torch, z)
    g = torch.zeros_like(zd)
    u = torch.zeros_like(zd)
    s.grad_g(zd, g, u)
    net = osolver.make_net(cfg, prob["weights"])
    for b in range(z.shape[0]):
        ref = net.grad_g(z[b].astype(np.float64))
        assert rel_l2(g[b].cpu().numpy(), ref) <= tol
        uref = net.N(z[b].astype(np.float64)) - z[b]
        assert rel_l2(u[b].cpu().numpy(), uref) <= tol


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_fidelity_component(name):
    torch = torch_cuda()
    cfg = _mini(name)
    prob = synth.make_problem(cfg)
    s = _solver(cfg, prob, "fp32")
    fids = osolver.make_fidelities(cfg, prob)
    x = prob["x_true"].astype(np.float32)
    if name == "C4":
        x = (0.9 * x + 0.05).astype(np.float32)   # away from the noise-free zero of grad f
    out = torch.zeros_like(_dev(torch, x))
    if name != "C5":
        s.fidelity_grad(_dev(torch, prob["y"]), _dev(torch, x), out)
        for b in range(x.shape[0]):
            assert rel_l2(out[b].cpu().numpy(), fids[b].grad(x[b].astype(np.float64))) <= 1e-5
    if name == "C5":
        s.fidelity_prox(_dev(torch, prob["y"]), _dev(torch, x), 0.7, out)
        for b in range(x.shape[0]):
            assert rel_l2(out[b].cpu().numpy(), fids[b].prox(x[b].astype(np.float64), 0.7)) <= 2e-6
    if cfg["op"] == "inpaint":
        s.fidelity_prox(_dev(torch, prob["y"]), _dev(torch, x), 0.7, out)
        for b in range(x.shape[0]):
            assert rel_l2(out[b].cpu().numpy(), fids[b].prox(x[b].astype(np.float64), 0.7)) <= 1e-6


def _run_pair(name, precision, K, lam=None, **kw):
    torch = torch_cuda()
    cfg = _mini(name, **kw)
    prob = synth.make_problem(cfg)
    s = _solver(cfg, prob, precision)
    p = s.params(lam=lam, max_iter=K, tol=0.0)
    yd = _dev(torch, prob["y"])
    xd = _dev(torch, prob["x0"])
    st, code, tr = s.solve(yd, xd, p, trace=True)
    orc = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0, lam=lam, trace=True)
    return cfg, prob, xd.cpu().numpy(), st, tr, orc


@pytest.mark.parametrize("name,K", [("C1", 100), ("C2", 10), ("C3", 10), ("C4", 10), ("C5", 10),
                                    ("C2", 50), ("C3", 50), ("C4", 50), ("C5s", 50)])
@pytest.mark.parametrize("stress", [False, True])
def test_trajectory_fp32(name, K, stress):
    """fp32 iterates after K steps within 1e-4 relative L2, residual within 1e-6 (north_star).
    The stress variant raises lambda so that lam*grad g is not negligible."""
    lam = None
    kw = {}
    if name == "C5s":  # K = 50 on a smaller C5 plane (U-Net-64: the oracle's cost)
        name, kw = "C5", dict(H=32, W=64)
    if stress:
        kw.update(init_scale=configs.STRESS[name]["init_scale"])
        lam = configs.STRESS[name]["lam"]
    cfg, prob, x, st, tr, orc = _run_pair(name, "fp32", K, lam=lam, **kw)
    assert (st["status"] == 1).all() and (st["iters"] == K).all()
    for b in range(x.shape[0]):
        assert rel_l2(x[b], orc["x"][b]) <= 1e-4
        assert abs(st["residual"][b] - orc["residual"][b]) <= 1e-6
    assert np.allclose(tr, orc["rmax_trace"], rtol=1e-3, atol=1e-6)


@pytest.mark.parametrize("name,kw", [("C2", dict(H=32, W=32)), ("C3", dict(H=32, W=32)), ("C4", dict()),
                                     ("C5", dict(H=32, W=32))])
def test_trajectory_fp32_max_iter(name, kw):
    """The whole horizon of each config (K = max_iter: 200 / 300 / 300 / 200 operator
    applications), fp32 mode, images 0 and N-1 of the reduced batch: iterates
    within 1e-4 relative L2 and residuals within 1e-6 of the oracle at the LAST step, and the
    max-residual trace along the way. Smaller planes than the K = 10 / 50 cases keep the fp64
    oracle's 200-300 iterations at about a minute per config."""
    K = configs.CONFIGS[name]["max_iter"]
    cfg, prob, x, st, tr, orc = _run_pair(name, "fp32", K, **kw)
    assert (st["status"] == 1).all() and (st["iters"] == K).all()
    for b in range(x.shape[0]):
        assert rel_l2(x[b], orc["x"][b]) <= 1e-4
        assert abs(st["residual"][b] - orc["residual"][b]) <= 1e-6
    assert np.allclose(tr, orc["rmax_trace"], rtol=1e-3, atol=1e-6)


@pytest.mark.parametrize("name,K", [("C2", 30), ("C3", 30), ("C4", 30), ("C5", 30)])
@pytest.mark.parametrize("stress", [False, True])
def test_trajectory_bf16_psnr(name, K, stress):
    """bf16 reconstruction PSNR within 0.05 dB of the oracle's (north_star). The stress variant
    (init x0.3 and a lambda with ||lam grad g(x0)|| >= 0.1 ||grad f||) makes the
    tcgen05 network a visible part of every step."""
    lam = None
    kw = {}
    if stress:
        kw = dict(init_scale=configs.STRESS[name]["init_scale"])
        lam = configs.STRESS[name]["lam"]
    cfg, prob, x, st, tr, orc = _run_pair(name, "bf16", K, lam=lam, **kw)
    for b in range(x.shape[0]):
        d = abs(psnr(x[b], prob["x_true"][b]) - psnr(orc["x"][b], prob["x_true"][b]))
        assert d <= 0.05, d


def test_stop_rule_per_image_matches_oracle():
    """tol = 1e-4 per-image stop: same stop iteration per image as the oracle."""
    torch = torch_cuda()
    cfg = _mini("C3", batch=3)
    prob = synth.make_problem(cfg)
    s = _solver(cfg, prob, "fp32")
    p = s.params(max_iter=60, tol=1e-4)
    xd = _dev(torch, prob["x0"])
    st, code, _ = s.solve(_dev(torch, prob["y"]), xd, p)
    orc = osolver.solve_config(cfg, prob, max_iter=60, tol=1e-4)
    for b in range(3):
        if abs(orc["residual"][b] - 1e-4) > 1e-6:
            assert st["iters"][b] == orc["iters"][b]
            assert st["status"][b] == orc["status"][b]
        assert rel_l2(xd[b].cpu().numpy(), orc["x"][b]) <= 1e-4


def test_divergence_freezes_image():
    """Reading Q22: a non-finite iterate marks the image diverged and keeps its last finite iterate;
    the other images are unaffected."""
    torch = torch_cuda()
    cfg = _mini("C3", batch=2)
    prob = synth.make_problem(cfg)
    s = _solver(cfg, prob, "fp32")
    x0 = prob["x0"].copy()
    x0[1, 0, 3, 3] = np.inf
    xd = _dev(torch, x0)
    st, code, _ = s.solve(_dev(torch, prob["y"]), xd, s.params(max_iter=5, tol=0.0))
    from paper_2605_19705_b200 import ideq
    assert code == ideq.E_DIVERGED
    assert st["status"][1] == 2 and st["iters"][1] == 0
    assert st["status"][0] == 1 and st["iters"][0] == 5
    assert np.isfinite(xd[0].cpu().numpy()).all()


def test_global_max_rule_with_nccl_single_rank():
    """GLOBAL_MAX (BASELINE C5): the check-iteration graph with the NCCL MAX all-reduce (a
    world-1 communicator on this one-GPU box) stops on the oracle's iteration and gives the
    same iterates as the run without a communicator, bit for bit."""
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    cfg = _mini("C5", check_every=3, tol=5e-3, max_iter=60)
    prob = synth.make_problem(cfg)
    orc = osolver.solve_config(cfg, prob)
    outs = []
    for use_nccl in (False, True):
        nid = ideq.nccl_unique_id() if use_nccl else None
        s = ideq.Solver(cfg, prob["weights"], precision="fp32", max_batch=2, rank=0, world=1, nccl_id=nid)
        s.set_operator(prob)
        xd = _dev(torch, prob["x0"])
        st, code, _ = s.solve(_dev(torch, prob["y"]), xd, s.params())
        outs.append((st, xd.cpu().numpy()))
        s.close()
    assert np.array_equal(outs[0][1], outs[1][1])
    for st, x in outs:
        assert (st["iters"] == orc["iters"]).all() and (st["status"] == orc["status"]).all()
        assert orc["status"][0] == 0 and orc["iters"][0] % 3 == 0
        for b in range(2):
            assert rel_l2(x[b], orc["x"][b]) <= 1e-4


def test_solve_host_matches_device():
    torch = torch_cuda()
    cfg = _mini("C3")
    prob = synth.make_problem(cfg)
    s = _solver(cfg, prob, "fp32")
    p = s.params(max_iter=5, tol=0.0)
    xd = _dev(torch, prob["x0"])
    s.solve(_dev(torch, prob["y"]), xd, p)
    xh = prob["x0"].astype(np.float32).copy()
    s.solve_host(prob["y"].astype(np.float32), xh, p)
    assert np.array_equal(xh, xd.cpu().numpy())


def test_determinism_and_batch_independence():
    """Per-image computation independent of batch position and size: the
    batch-of-3 result for image 2 equals the batch-of-1 result bit for bit."""
    torch = torch_cuda()
    cfg = _mini("C3", batch=3)
    prob = synth.make_problem(cfg)
    for precision in ("fp32", "bf16"):
        s = _solver(cfg, prob, precision)
        p = s.params(max_iter=6, tol=0.0)
        xa = _dev(torch, prob["x0"])
        s.solve(_dev(torch, prob["y"]), xa, p)
        xb = _dev(torch, prob["x0"])
        s.solve(_dev(torch, prob["y"]), xb, p)
        assert torch.equal(xa, xb)
        sub = synth.make_problem(cfg, images=[2])
        s1 = _solver(cfg, sub, precision)
        x1 = _dev(torch, sub["x0"])
        s1.solve(_dev(torch, sub["y"]), x1, s1.params(max_iter=6, tol=0.0))
        assert torch.equal(x1[0], xa[2])


@pytest.mark.parametrize("ks,H,W", [(25, 64, 96), (9, 72, 64), (15, 64, 80), (15, 128, 72), (7, 48, 40), (9, 32, 40)])
def test_direct_blur_kernel_sizes(ks, H, W):
    """Direct-blur gradient step at every register-blocked kernel size (9, 15 -- C2's, at >= 64 x 64
    planes so the register-blocked kernel runs --, 25) and
    the 32-tile kernel (size 7, and planes smaller than 64 x 64): grad f component within 1e-5 and an fp32 trajectory within 1e-4 / 1e-6
    (C5 geometry with the gradient variant; 64 x 64 blur tiles with ragged edges)."""
    torch = torch_cuda()
    cfg = _mini("C5", H=H, W=W, step="grad", blur_impl="direct", ksize=ks, ksigma=ks / 8.0)
    prob = synth.make_problem(cfg)
    s = _solver(cfg, prob, "fp32")
    fids = osolver.make_fidelities(cfg, prob)
    # away from the truth: at x_true, A^T(Ax - y) = -A^T n is the noise smoothed by the kernel
    # (|.| ~ sigma / k), and the fp32 rounding of Ax (~1e-7 |Ax|) is then 1e-5..1e-4 of it
    x = (0.9 * prob["x_true"] + 0.05).astype(np.float32)
    out = torch.zeros_like(_dev(torch, x))
    s.fidelity_grad(_dev(torch, prob["y"]), _dev(torch, x), out)
    for b in range(x.shape[0]):
        assert rel_l2(out[b].cpu().numpy(), fids[b].grad(x[b].astype(np.float64))) <= 1e-5
    K = 6
    xd = _dev(torch, prob["x0"])
    st, code, _ = s.solve(_dev(torch, prob["y"]), xd, s.params(max_iter=K, tol=0.0))
    orc = osolver.solve_config(cfg, prob, max_iter=K, tol=0.0)
    xg = xd.cpu().numpy()
    for b in range(xg.shape[0]):
        assert rel_l2(xg[b], orc["x"][b]) <= 1e-4
        assert abs(st["residual"][b] - orc["residual"][b]) <= 1e-6


@pytest.mark.parametrize("batch,tol,K,H", [(1, 0.0, 100, 32), (3, 0.0, 40, 32), (3, 5e-4, 200, 32),
                                           (2, 0.0, 30, 16), (2, 5e-4, 200, 64)])
def test_tiny_whole_solve_kernel(batch, tol, K, H):
    """C1's whole solve in one launch (tiny_solve.cu: one cluster per image, DSMEM halos; H = 32
    and 64 run 16-CTA clusters of 2 / 4 rows (the 9x9 blur halo reaches two CTAs up and down at
    2 rows), H = 16 an 8-CTA cluster of 2 rows): fp32 iterates within 1e-4 and residuals within 1e-6
    of the oracle, stop iterations equal (tol > 0, per-image rule), and the same result as the
    per-iteration kernels (the profiling mode launches those eagerly) within fp32 rounding."""
    torch = torch_cuda()
    cfg = _mini("C1", batch=batch, H=H)
    prob = synth.make_problem(cfg)
    orc = osolver.solve_config(cfg, prob, max_iter=K, tol=tol, trace=True)
    s = _solver(cfg, prob, "fp32")
    outs = []
    for prof in (False, True):
        s.set_profiling(prof)
        xd = _dev(torch, prob["x0"])
        st, code, tr = s.solve(_dev(torch, prob["y"]), xd, s.params(max_iter=K, tol=tol), trace=True)
        assert (s.launches_per_iteration() == 0) == (not prof)   # fused <=> one launch per solve
        outs.append((st, xd.cpu().numpy(), tr))
    for st, x, tr in outs:
        assert np.array_equal(st["iters"], orc["iters"]) and np.array_equal(st["status"], orc["status"])
        for b in range(batch):
            assert rel_l2(x[b], orc["x"][b]) <= 1e-4
            assert abs(st["residual"][b] - orc["residual"][b]) <= 1e-6
        n = int(orc["iters"].max())
        assert np.allclose(tr[:n], orc["rmax_trace"][:n], rtol=1e-3, atol=1e-6)
    assert rel_l2(outs[0][1], outs[1][1]) <= 1e-5


@pytest.mark.parametrize("name,H,W,batch", [("C4", 256, 256, 16), ("C4", 512, 256, 2), ("C4", 128, 512, 2),
                                            ("C5", 512, 512, 2), ("C5", 256, 512, 2), ("C5", 512, 128, 2),
                                            ("C5", 256, 256, 3)])
def test_fft_operators_at_register_fft_sizes(name, H, W, batch):
    """The register-resident FFT passes (N = 256 / 512 along either axis, mixed with the shared-
    memory passes for other sizes): phase-retrieval gradient (C4, P:958-970 style unitary F) and
    FFT blur prox (C5) against the oracle's numpy FFT definitions, per image."""
    torch = torch_cuda()
    kw = dict(H=H, W=W, batch=batch)
    if name == "C4":
        kw["tau"] = 0.5 / 17
    cfg = configs.get(name, **kw)
    prob = synth.make_problem(cfg)
    s = _solver(cfg, prob, "fp32")
    fids = osolver.make_fidelities(cfg, prob)
    x = (0.9 * prob["x_true"] + 0.05).astype(np.float32)
    out = torch.zeros_like(_dev(torch, x))
    if name == "C4":
        s.fidelity_grad(_dev(torch, prob["y"]), _dev(torch, x), out)
        for b in range(batch):
            assert rel_l2(out[b].cpu().numpy(), fids[b].grad(x[b].astype(np.float64))) <= 1e-5, b
    else:
        s.fidelity_prox(_dev(torch, prob["y"]), _dev(torch, x), 0.7, out)
        for b in range(batch):
            assert rel_l2(out[b].cpu().numpy(), fids[b].prox(x[b].astype(np.float64), 0.7)) <= 2e-6, b


@pytest.mark.parametrize("J,H", [(4, 256), (2, 256), (1, 8), (3, 256)])
def test_phase_gradient_mask_counts(J, H):
    """Phase-retrieval gradient with J masks (the register row pass sums the J inverse rows of a
    pixel in a fixed order; J not dividing 16 takes the shared-memory pass) at W = 256."""
    torch = torch_cuda()
    cfg = configs.get("C4", batch=2, H=H, W=256, n_phase=J, tau=0.5 / 17)
    prob = synth.make_problem(cfg)
    s = _solver(cfg, prob, "fp32")
    fids = osolver.make_fidelities(cfg, prob)
    x = (0.9 * prob["x_true"] + 0.05).astype(np.float32)
    out = torch.zeros_like(_dev(torch, x))
    s.fidelity_grad(_dev(torch, prob["y"]), _dev(torch, x), out)
    for b in range(2):
        assert rel_l2(out[b].cpu().numpy(), fids[b].grad(x[b].astype(np.float64))) <= 1e-5, b
