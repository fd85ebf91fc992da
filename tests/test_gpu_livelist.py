"""Early-stopping solves through the live-image list (stop rule PAPER P:796 and
P:860, reading Q17): once an image's relative residual reaches tol it is frozen, and every
network kernel walks only the tiles of the images still active (include/ideq.h,
ideq_params.compute_frozen).

- on/off: the same solve with the list switched off (compute_frozen = 1) gives the same
  per-image stop iterations, residuals and iterates, bit for bit (frozen images are never
  written either way);
- oracle: each image's stop iteration is consistent with the fp64 oracle's residual trace under a
  perturbation of r (fp32: 1e-6 absolute; bf16: 5% of tol, reading B1 in
  DESIGN.md -- the bf16 network moves r by up to a few percent, and where r is flat near tol
  that moves the stop by several iterations), and the iterates agree at that iteration (fp32:
  1e-4 relative L2; bf16: the north_star's 0.05 dB PSNR bar);
- full size (C3, 32 x 3 x 256 x 256, the bench's launch configuration): sampled images {0, 31}
  against the oracle's early-stopping solve of those images (tests/golden/c3_stop_oracle.npz,
  written by tools/make_golden_c3_stop.py from oracle/ only);
- more than 1024 images (the list is built in chunks of the bookkeeping block).
"""
import os

import numpy as np
import pytest

from oracle import solver as osolver
from paper_2605_19705_b200 import configs, synth
from tests.gpu_util import psnr, rel_l2, torch_cuda

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c3_stop_oracle.npz")
BAND = 0.05  # bf16 near-tie band on the oracle's residual (reading B1)


def _solve(cfg, prob, precision, **pk):
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    s = ideq.Solver(cfg, prob["weights"], precision=precision, max_batch=cfg["batch"])
    s.set_operator(prob)
    xd = torch.tensor(np.ascontiguousarray(prob["x0"], dtype=np.float32)).cuda()
    yd = torch.tensor(np.ascontiguousarray(prob["y"], dtype=np.float32)).cuda()
    st, code, _ = s.solve(yd, xd, s.params(**pk))
    x = xd.cpu().numpy()
    s.close()
    return st, x


def oracle_trace(cfg, prob, b, K, lam, x0, capture):
    """The oracle's iteration of image b alone (osolver.ideq_step, Eq. 6 / Alg. 2) for K steps with
    tol = 0: its residual after every update (trace[k] = r after update k + 1) and the iterates
    after the updates listed in `capture`."""
    sub = synth.make_problem(cfg, images=[b])
    net = osolver.make_net(cfg, sub["weights"])
    fid = osolver.make_fidelities(cfg, sub)[0]
    x = np.asarray(x0, dtype=np.float64)
    xp = x.copy()
    trace, xs = [], {}
    for k in range(K):
        xn = osolver.ideq_step(x, xp, net, fid, lam, cfg["tau"], cfg["beta"], cfg["step"])
        trace.append(osolver.residual(xn, x))
        xp, x = x, xn
        if k + 1 in capture:
            xs[k + 1] = x.copy()
    return np.array(trace), xs


def stop_consistent(k_gpu, trace, tol, K, d_rel=0.0, d_abs=0.0):
    """The per-image rule stops at the first k with r_k <= tol (reading Q17). A stop iteration is
    consistent with the oracle's residual trace under a perturbation of r by at most
    d = d_rel * tol + d_abs when r at the stop is <= tol + d (or the cap was hit with every r
    above tol - d) and every earlier r is > tol - d."""
    d = d_rel * tol + d_abs
    k = int(k_gpu)
    earlier_ok = all(r > tol - d for r in trace[:k - 1])
    if k == K and trace[K - 1] > tol - d:
        return earlier_ok
    return earlier_ok and trace[k - 1] <= tol + d


def _assert_same(a, b):
    for key in ("iters", "status", "residual"):
        assert np.array_equal(a[0][key], b[0][key]), key
    assert np.array_equal(a[1], b[1])


def test_live_list_on_off_bitwise_fullsize_c3():
    """C3 at its full per-GPU size, bf16, tol = 1e-4 (the bench's ms-to-tolerance solve)."""
    cfg = configs.get("C3")
    prob = synth.make_problem(cfg)
    on = _solve(cfg, prob, "bf16", tol=1e-4)
    off = _solve(cfg, prob, "bf16", tol=1e-4, compute_frozen=True)
    _assert_same(on, off)
    st = on[0]
    # with the random-init network some images reach tol at once (r_1 <= 1e-4) and freeze while
    # the others run on: the list shrinks and the remaining tiles are re-balanced
    assert (st["status"] == 0).any() and (st["iters"] < cfg["max_iter"]).any(), "no image stopped early"
    assert (st["iters"] == cfg["max_iter"]).any(), "no image ran on"


_ORC = {}


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_live_list_stop_iterations_match_oracle(precision):
    """Reduced C3 (6 images of 3 x 32 x 32; level 3 is 4 x 4), started from the flat image 0.5
    with lambda = 0.3 and tol = 1e-3: the images stop at different iterations, some hit the cap,
    so the live list shrinks in steps. Every image: its stop iteration is consistent with the
    oracle's residual trace (fp32: |delta r| <= 1e-6; bf16: 5% of tol, reading
    B1) and its iterate matches the oracle's at that iteration (fp32 1e-4 rel. L2; bf16 0.05 dB)."""
    cfg = configs.get("C3", batch=6, H=32, W=32)
    prob = synth.make_problem(cfg)
    prob["x0"] = np.full_like(prob["x0"], 0.5)
    tol, K, lam = 1e-3, 120, 0.3
    st, x = _solve(cfg, prob, precision, lam=lam, tol=tol, max_iter=K)
    off = _solve(cfg, prob, precision, lam=lam, tol=tol, max_iter=K, compute_frozen=True)
    _assert_same((st, x), off)
    assert len(set(st["iters"].tolist())) >= 3, st["iters"]
    for b in range(cfg["batch"]):
        kg = int(st["iters"][b])
        if b not in _ORC:  # the oracle's trajectory of image b (shared by both precisions)
            _ORC[b] = oracle_trace(cfg, prob, b, K, lam, prob["x0"][b], set(range(1, K + 1)))
        tr, xs = _ORC[b]
        if precision == "bf16":
            assert stop_consistent(kg, tr, tol, K, d_rel=BAND), (b, kg, tr[max(kg - 3, 0):kg + 2])
            d = abs(psnr(x[b], prob["x_true"][b]) - psnr(xs[kg], prob["x_true"][b]))
            assert d <= 0.05, (b, d)
        else:
            assert stop_consistent(kg, tr, tol, K, d_abs=1e-6), (b, kg, tr[max(kg - 3, 0):kg + 2])
            assert rel_l2(x[b], xs[kg]) <= 1e-4, b
        # stopped before the cap => converged; at the cap either status is consistent with the trace
        if kg < K:
            assert st["status"][b] == 0, b
        else:
            d = BAND * tol if precision == "bf16" else 1e-6
            assert (st["status"][b] == 0 and tr[K - 1] <= tol + d) or (st["status"][b] == 1 and tr[K - 1] > tol - d), b


@pytest.mark.skipif(not os.path.exists(GOLD), reason="golden oracle solve not generated")
def test_live_list_fullsize_c3_sampled_vs_oracle():
    """Full-size C3, bf16, tol = 1e-4, per-image rule (the bench's ms-to-tolerance solve): the
    sampled images stop where the oracle's residual trace allows (reading B1) and reconstruct
    within 0.05 dB of the oracle's iterate at its own stop."""
    g = np.load(GOLD)
    cfg = configs.get("C3")
    prob = synth.make_problem(cfg)
    st, x = _solve(cfg, prob, "bf16", tol=1e-4)
    K = cfg["max_iter"]
    for i in g["images"]:
        tr = g[f"rtrace_{i}"]
        kg = int(st["iters"][i])
        assert kg <= len(tr) or len(tr) == K, (i, kg, len(tr))
        assert stop_consistent(kg, tr, 1e-4, K, d_rel=BAND), (i, kg, int(g[f"iters_{i}"]))
        xo = g[f"x_{i}"].astype(np.float64)
        d = abs(psnr(x[i], prob["x_true"][i]) - psnr(xo, prob["x_true"][i]))
        assert d <= 0.05, (i, d)


def test_live_list_more_than_1024_images():
    """1100 images of 3 x 16 x 16: the bookkeeping block builds the compacted list in chunks of
    1024. The list on/off solves agree bit for bit, and the last images equal a separate solve of
    those images alone (per-image results do not depend on the batch)."""
    cfg = configs.get("C3", batch=1100, H=16, W=16)
    prob = synth.make_problem(cfg)
    prob["x0"] = np.full_like(prob["x0"], 0.5)   # varied stop iterations (as in the test above)
    pk = dict(lam=0.3, tol=1e-3, max_iter=60)
    on = _solve(cfg, prob, "bf16", **pk)
    off = _solve(cfg, prob, "bf16", compute_frozen=True, **pk)
    _assert_same(on, off)
    its = on[0]["iters"]
    assert (its < 60).sum() > 100 and len(set(its.tolist())) >= 2, sorted(set(its.tolist()))
    idx = list(range(1090, 1100))
    cfg_s = configs.get("C3", batch=len(idx), H=16, W=16)
    sub = synth.make_problem(cfg_s, images=idx)
    sub["x0"] = np.full_like(sub["x0"], 0.5)
    st_s, x_s = _solve(cfg_s, sub, "bf16", **pk)
    assert np.array_equal(st_s["iters"], on[0]["iters"][idx])
    assert np.array_equal(x_s, on[1][idx])


def test_solve_batch_above_operator_batch_rejected():
    """The operator's per-image data and FFT work spectrum are sized by set_operator's batch:
    a larger solve is refused (IDEQ_E_INVALID), for every operator kind."""
    torch = torch_cuda()
    from paper_2605_19705_b200 import ideq
    for name, kw in (("C3", dict(H=32, W=32)), ("C5", dict(H=32, W=32)), ("C4", dict(H=32, W=32, tau=0.5 / 21))):
        cfg = configs.get(name, batch=3, **kw)
        prob = synth.make_problem(cfg)
        s = ideq.Solver(cfg, prob["weights"], precision="bf16", max_batch=3)
        s.set_operator(prob, batch=2)
        y = torch.tensor(prob["y"].astype(np.float32)).cuda()
        x = torch.tensor(prob["x0"].astype(np.float32)).cuda()
        with pytest.raises(ideq.IdeqError) as ei:
            s.solve(y, x, s.params(max_iter=2, tol=0.0))
        assert ei.value.code == ideq.E_INVALID, name
        s.close()
