"""Oracle i-DEQ inference loop (fp64), Algorithms 1 and 2 of the paper with frozen Theta.

Per image i (images are independent except under the global-max stop rule):
  x^{-1} = x^0                                           P:210 / P:632
  repeat for k = 0 .. max_iter-1 while active:
    z^k     = x^k + beta (x^k - x^{k-1})                 Eq. 4, beta = 1 - alpha (Q1)
    grad    : x^{k+1} = z^k - tau (grad f(z^k) + lam grad g(z^k))      Alg. 1 l.8
    prox    : x^{k+1} = prox_{tau f}(z^k - tau lam grad g(z^k))        Alg. 2 l.7
    r       = ||x^{k+1} - x^k|| / ||x^k||                P:796, P:860 (reading Q3)
    non-finite x^{k+1}: status diverged, keep x^k        reading Q22
    per_image : stop image when (k+1) % C == 0 and r <= tol            reading Q17
    global_max: stop all when (k+1) % C == 0 and max_active r <= tol   BASELINE C5
  output x_hat = last accepted iterate (Remark 1; no averaging, no restart, Q4/Q5)

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

from .nets import Net
from .operators import Fidelity

CONVERGED, MAX_ITER, DIVERGED = 0, 1, 2


def ideq_step(x, x_prev, net, fid, lam, tau, beta, step):
    """One application of T^{i-DEQ} (Eq. 6) or T^{i-DEQ-P}."""
    z = x + beta * (x - x_prev)                                   # inertial step, Eq. 4
    gg = net.grad_g(z)
    if step == "grad":
        return z - tau * (fid.grad(z) + lam * gg)                 # Alg. 1 l.8
    return fid.prox(z - tau * lam * gg, tau)                      # Alg. 2 l.7


def residual(x_new, x_old):
    """||x^{k+1} - x^k||_2 / ||x^k||_2 over all C*H*W entries; +inf if ||x^k|| = 0 (Q3)."""
    num = float(np.sqrt(np.sum((x_new - x_old) ** 2)))
    den = float(np.sqrt(np.sum(x_old ** 2)))
    return num / den if den > 0 else float("inf")


def make_net(cfg, weights):
    return Net(cfg["net"], weights, cfg["C"], cfg["widths"], cfg.get("identity_skip", True),
               cfg.get("act", "softplus"), cfg.get("res_blocks", 2))


def make_fidelities(cfg, prob):
    """One Fidelity per image of the problem dict built by synth.make_problem."""
    fids = []
    for b in range(len(prob["images"])):
        if cfg["op"] == "blur":
            k = prob["kernels"][b] if cfg.get("kernel_per_image", False) else prob["kernel"]
            fids.append(Fidelity("blur", prob["y"][b], kernel=k))
        elif cfg["op"] == "inpaint":
            fids.append(Fidelity("inpaint", prob["y"][b], mask=prob["masks"][b]))
        else:
            fids.append(Fidelity("phase", prob["y"][b], phase=prob["phase_masks"]))
    return fids


def solve(net, fids, x0, lam, tau, beta, max_iter, tol, step="grad", check_every=1,
          stop_rule="per_image", trace=False):
    """Run the batched loop. x0: [B][C][H][W] (promoted to float64).
    Returns dict(x, iters, residual, status[, rmax_trace])."""
    x0 = np.asarray(x0, dtype=np.float64)
    B = x0.shape[0]
    xc = [x0[b].copy() for b in range(B)]
    xp = [x0[b].copy() for b in range(B)]                         # x^{-1} = x^0
    active = [True] * B
    iters = [0] * B
    res = [float("nan")] * B
    status = [MAX_ITER] * B
    rtrace = []
    for k in range(max_iter):
        if not any(active):
            break
        r_now = []
        for b in range(B):
            if not active[b]:
                continue
            xn = ideq_step(xc[b], xp[b], net, fids[b], lam, tau, beta, step)
            r = residual(xn, xc[b])
            if not np.all(np.isfinite(xn)):
                status[b] = DIVERGED
                active[b] = False
                continue
            xp[b], xc[b] = xc[b], xn
            iters[b] = k + 1
            res[b] = r
            r_now.append(r)
        if trace:
            rtrace.append(max(r_now) if r_now else float("nan"))
        if (k + 1) % check_every == 0:
            if stop_rule == "per_image":
                for b in range(B):
                    if active[b] and res[b] <= tol:
                        active[b] = False
                        status[b] = CONVERGED
            else:
                act = [b for b in range(B) if active[b]]
                if act and max(res[b] for b in act) <= tol:
                    for b in act:
                        active[b] = False
                        status[b] = CONVERGED
    out = dict(x=np.stack(xc), iters=np.array(iters), residual=np.array(res),
               status=np.array(status))
    if trace:
        out["rmax_trace"] = np.array(rtrace)
    return out


def solve_config(cfg, prob, max_iter=None, tol=None, lam=None, trace=False):
    """Convenience wrapper: the oracle on a synth.make_problem dict."""
    net = make_net(cfg, prob["weights"])
    fids = make_fidelities(cfg, prob)
    return solve(net, fids, prob["x0"], cfg["lam"] if lam is None else lam, cfg["tau"], cfg["beta"],
                 cfg["max_iter"] if max_iter is None else max_iter,
                 cfg["tol"] if tol is None else tol, cfg["step"], cfg["check_every"],
                 cfg["stop_rule"], trace=trace)
