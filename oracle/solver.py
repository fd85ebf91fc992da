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
  output x_hat = last accepted iterate (Remark 1) unless averaging is on

Optional (readings R4, R5):
  restart (Eq. 5): after each accepted step, k_r += 1, S += ||x^{k+1} - x^k||^2;
    if k_r * S > B^2 the inertia is reset: the previous iterate is set to x^{k+1} (so the next
    z = x^{k+1}).  restart = 1: Alg. 1 semantics ("x^{-1}, x^0 <- x^k, k <- 0": k_r and
    S reset too); restart = 2: Alg. 2 semantics ("x^{k-1} <- x^k" only).
  averaging (Alg. 1/2 steps 12-13, P:232-237 / P:654-659): K0 = argmin over the global
    iteration index floor(K/2) < k < K-1 of ||x^{k+1} - x^k|| (first minimum), x_hat =
    mean(z^0 .. z^{K0}); empty window -> x_hat = x^K. Fixed-count solves only (tol = 0).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

from .nets import Net
from .operators import Fidelity

CONVERGED, MAX_ITER, DIVERGED = 0, 1, 2


def extrapolate(x, x_prev, beta):
    """z = x + (1 - alpha)(x - x_prev), Eq. 4; beta = 1 - alpha (Q1)."""
    return x + beta * (x - x_prev)


def red_step(z, net, fid, lam, tau, step):
    """T^{RED} (Eq. 3) or T^{RED-P} applied at z."""
    gg = net.grad_g(z)
    if step == "grad":
        return z - tau * (fid.grad(z) + lam * gg)                 # Alg. 1 l.8
    return fid.prox(z - tau * lam * gg, tau)                      # Alg. 2 l.7


def ideq_step(x, x_prev, net, fid, lam, tau, beta, step):
    """One application of T^{i-DEQ} (Eq. 6) or T^{i-DEQ-P}."""
    return red_step(extrapolate(x, x_prev, beta), net, fid, lam, tau, step)


def restart_check(k_since, inc_sq_sum, B):
    """Eq. 5: k * sum_{t<k} ||x^{t+1} - x^t||^2 > B^2."""
    return k_since * inc_sq_sum > B * B


def averaging_select(z_hist, incr, K):
    """Alg. 1 steps 12-13: K0 = argmin_{floor(K/2) < k < K-1} ||x^{k+1} - x^k||
    (first minimum), x_hat = (1 / (K0 + 1)) sum_{k=0}^{K0} z^k. Returns (K0, x_hat), or
    (None, None) when the window is empty (caller falls back to x^K)."""
    ks = list(range(K // 2 + 1, K - 1))
    if not ks:
        return None, None
    K0 = min(ks, key=lambda k: (incr[k], k))
    return K0, np.mean(np.stack(z_hist[:K0 + 1]), axis=0)


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
        elif cfg["op"] == "mri":
            fids.append(Fidelity("mri", prob["y"][b], mask=prob["kmask"]))
        elif cfg["op"] == "rician":
            fids.append(Fidelity("rician", prob["y"][b], sigma=cfg["sigma"]))
        else:
            fids.append(Fidelity("phase", prob["y"][b], phase=prob["phase_masks"]))
    return fids


def solve(net, fids, x0, lam, tau, beta, max_iter, tol, step="grad", check_every=1,
          stop_rule="per_image", trace=False, restart=0, restart_B=float("inf"), averaging=False):
    """Run the batched loop. x0: [B][C][H][W] (promoted to float64).
    Returns dict(x, iters, residual, status, restarts, k0[, rmax_trace])."""
    if averaging and tol > 0:
        raise ValueError("averaging is defined for fixed-count solves (tol = 0)")
    x0 = np.asarray(x0, dtype=np.float64)
    B = x0.shape[0]
    xc = [x0[b].copy() for b in range(B)]
    xp = [x0[b].copy() for b in range(B)]                         # x^{-1} = x^0
    active = [True] * B
    iters = [0] * B
    res = [float("nan")] * B
    status = [MAX_ITER] * B
    k_since = [0] * B                                             # Eq. 5 counter
    inc_sum = [0.0] * B                                           # Eq. 5 sum of ||x^{t+1}-x^t||^2
    restarts = [0] * B
    z_hist = [[] for _ in range(B)]
    incr = [[] for _ in range(B)]
    rtrace = []
    for k in range(max_iter):
        if not any(active):
            break
        r_now = []
        for b in range(B):
            if not active[b]:
                continue
            z = extrapolate(xc[b], xp[b], beta)                   # Eq. 4
            xn = red_step(z, net, fids[b], lam, tau, step)
            r = residual(xn, xc[b])
            if not np.all(np.isfinite(xn)):
                status[b] = DIVERGED
                active[b] = False
                continue
            inc2 = float(np.sum((xn - xc[b]) ** 2))
            if averaging:
                z_hist[b].append(z)
                incr[b].append(np.sqrt(inc2))
            k_since[b] += 1
            inc_sum[b] += inc2
            if restart and restart_check(k_since[b], inc_sum[b], restart_B):
                xp[b], xc[b] = xn, xn                             # inertia reset: next z = x^{k+1}
                restarts[b] += 1
                if restart == 1:                                  # Alg. 1: k <- 0
                    k_since[b], inc_sum[b] = 0, 0.0
            else:
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
    k0 = [-1] * B
    if averaging:
        for b in range(B):
            if status[b] != DIVERGED and iters[b] == max_iter:
                K0, xh = averaging_select(z_hist[b], incr[b], max_iter)
                if K0 is not None:
                    k0[b] = K0
                    xc[b] = xh
    out = dict(x=np.stack(xc), iters=np.array(iters), residual=np.array(res),
               status=np.array(status), restarts=np.array(restarts), k0=np.array(k0))
    if trace:
        out["rmax_trace"] = np.array(rtrace)
    return out


def solve_config(cfg, prob, max_iter=None, tol=None, lam=None, trace=False, restart=0, restart_B=float("inf"),
                 averaging=False):
    """Convenience wrapper: the oracle on a synth.make_problem dict."""
    net = make_net(cfg, prob["weights"])
    fids = make_fidelities(cfg, prob)
    return solve(net, fids, prob["x0"], cfg["lam"] if lam is None else lam, cfg["tau"], cfg["beta"],
                 cfg["max_iter"] if max_iter is None else max_iter,
                 cfg["tol"] if tol is None else tol, cfg["step"], cfg["check_every"],
                 cfg["stop_rule"], trace=trace, restart=restart, restart_B=restart_B, averaging=averaging)
