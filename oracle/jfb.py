"""Oracle JFB training gradient at the fixed point, fp64.

Jacobian-free backpropagation: the loss is taken after ONE more
application of the i-DEQ operator at the (stopped) fixed point x_hat, treating x_hat as a
constant:  L = 1/2 sum_i ||T_Theta(x_hat_i) - x*_i||^2,  with x^{k-1} = x^k = x_hat so that the
extrapolation is z = x_hat (and dL/dbeta = 0).

  gradient step (Alg. 1 l.8):  T = z - tau (grad f(z) + lam grad g_theta(z))
  prox step (Alg. 2 l.7):      T = prox_{tau f}(z - tau lam grad g_theta(z))   (inpainting only:
                               its closed form has the diagonal Jacobian 1 / (1 + tau M))

With the identity skip, grad g_theta(z) = J_U(z)^T U(z), so for a cotangent v
  <v, grad g> = <J_U(z) v, U(z)> = <U'(z)[v], U(z)>          (adjoint identity)
and dL/dtheta = -tau lam d/dtheta <v, grad g_theta(z)> with v = r = T - x* (gradient step) or
v = r / (1 + tau M) (prox). The theta-derivative of <U'(z)[v], U(z)> is computed by running the
network forward on the primal z AND the tangent v (forward-mode: same linear layers; softplus
tangent sp'(p) p_dot), then one reverse pass over both streams: every linear layer passes both
cotangents through its adjoint and collects the weight gradient of both streams; softplus gives
  p_dot_bar = sp'(p) a_dot_bar,  p_bar = sp'(p) a_bar + sp''(p) p_dot a_dot_bar,
  sp'(p) = sigmoid(p), sp''(p) = sp'(p) (1 - sp'(p)).
Seeds: U_bar = U_dot, U_dot_bar = U.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

from . import nets


def _sp(p):
    return nets.softplus(p)


def _s1(p):
    return nets.softplus_grad(p)


def _wgrad3(x, g):
    """d/dW of <g, conv3x3(x, W)>: dW[co,ci,a,b] = sum_{m,n} g[co,m,n] x[ci, m+a-1, n+b-1]."""
    Cin, H, Wd = x.shape
    xp = np.zeros((Cin, H + 2, Wd + 2))
    xp[:, 1:H + 1, 1:Wd + 1] = x
    g2 = g.reshape(g.shape[0], -1)
    dW = np.zeros((g.shape[0], Cin, 3, 3))
    for a in range(3):
        for b in range(3):
            dW[:, :, a, b] = g2 @ xp[:, a:a + H, b:b + Wd].reshape(Cin, -1).T
    return dW


def _wgrad_down(x, g):
    """d/dWd of <g, down2x2(x, Wd)>: dWd[co,ci,a,b] = sum_{i,j} g[co,i,j] x[ci, 2i+a, 2j+b]."""
    Cin = x.shape[0]
    g2 = g.reshape(g.shape[0], -1)
    dW = np.zeros((g.shape[0], Cin, 2, 2))
    for a in range(2):
        for b in range(2):
            dW[:, :, a, b] = g2 @ x[:, a::2, b::2].reshape(Cin, -1).T
    return dW


def _wgrad_up(x, g):
    """d/dWu of <g, up2x2(x, Wu)>: dWu[ci,co,a,b] = sum_{i,j} x[ci,i,j] g[co, 2i+a, 2j+b]."""
    Cin = x.shape[0]
    x2 = x.reshape(Cin, -1)
    dW = np.zeros((Cin, g.shape[0], 2, 2))
    for a in range(2):
        for b in range(2):
            dW[:, :, a, b] = x2 @ g[:, a::2, b::2].reshape(g.shape[0], -1).T
    return dW


def phi_weight_grad(net, z, v):
    """d/dtheta <v, grad g_theta(z)> for a Net with identity skip, as a dict name -> dW."""
    if not net.identity_skip:
        raise ValueError("the JFB oracle assumes the identity skip N = z + U (all BASELINE nets)")
    W, R = net.W, net.res_blocks
    dW = {k: np.zeros_like(w) for k, w in W.items()}
    if net.arch == "tiny3":
        # forward: p1 = c1 z, a1 = sp(p1), p2 = c2 a1, a2 = sp(p2), U = c3 a2 ; tangent alike
        p1 = nets.conv3x3(z, W["c1"]); a1 = _sp(p1)
        p2 = nets.conv3x3(a1, W["c2"]); a2 = _sp(p2)
        U = nets.conv3x3(a2, W["c3"])
        p1d = nets.conv3x3(v, W["c1"]); a1d = _s1(p1) * p1d
        p2d = nets.conv3x3(a1d, W["c2"]); a2d = _s1(p2) * p2d
        Ud = nets.conv3x3(a2d, W["c3"])
        Ub, Udb = Ud, U
        dW["c3"] += _wgrad3(a2, Ub) + _wgrad3(a2d, Udb)
        a2b, a2db = nets.conv3x3_T(Ub, W["c3"]), nets.conv3x3_T(Udb, W["c3"])
        p2db = _s1(p2) * a2db
        p2b = _s1(p2) * a2b + _s1(p2) * (1 - _s1(p2)) * p2d * a2db
        dW["c2"] += _wgrad3(a1, p2b) + _wgrad3(a1d, p2db)
        a1b, a1db = nets.conv3x3_T(p2b, W["c2"]), nets.conv3x3_T(p2db, W["c2"])
        p1db = _s1(p1) * a1db
        p1b = _s1(p1) * a1b + _s1(p1) * (1 - _s1(p1)) * p1d * a1db
        dW["c1"] += _wgrad3(z, p1b) + _wgrad3(v, p1db)
        return dW

    # ---- U-Net: forward of both streams with a tape
    tape = []                       # (kind, name, x, x_dot[, p, p_dot]) in forward order
    t = nets.conv3x3(z, W["head"]); td = nets.conv3x3(v, W["head"])
    tape.append(("head", "head", z, v))
    skips = {}
    for l in range(4):
        for r in range(R):
            nA, nB = f"e{l}.{r}.A", f"e{l}.{r}.B"
            p = nets.conv3x3(t, W[nA]); pd = nets.conv3x3(td, W[nA])
            a = _sp(p); ad = _s1(p) * pd
            tape.append(("rb", (nA, nB), t, td, p, pd, a, ad))
            t = t + nets.conv3x3(a, W[nB]); td = td + nets.conv3x3(ad, W[nB])
        if l < 3:
            skips[l] = (t, td)
            tape.append(("down", f"down{l}", t, td))
            t = nets.down2x2(t, W[f"down{l}"]); td = nets.down2x2(td, W[f"down{l}"])
    for l in (2, 1, 0):
        tape.append(("up", f"up{l}", t, td, l))
        t = nets.up2x2(t, W[f"up{l}"]) + skips[l][0]
        td = nets.up2x2(td, W[f"up{l}"]) + skips[l][1]
        for r in range(R):
            nA, nB = f"d{l}.{r}.A", f"d{l}.{r}.B"
            p = nets.conv3x3(t, W[nA]); pd = nets.conv3x3(td, W[nA])
            a = _sp(p); ad = _s1(p) * pd
            tape.append(("rb", (nA, nB), t, td, p, pd, a, ad))
            t = t + nets.conv3x3(a, W[nB]); td = td + nets.conv3x3(ad, W[nB])
    U = nets.conv3x3(t, W["tail"]); Ud = nets.conv3x3(td, W["tail"])

    # ---- reverse over both streams: seeds U_bar = U_dot, U_dot_bar = U
    gb, gdb = Ud, U
    dW["tail"] += _wgrad3(t, gb) + _wgrad3(td, gdb)
    gb, gdb = nets.conv3x3_T(gb, W["tail"]), nets.conv3x3_T(gdb, W["tail"])
    skip_bar = {}
    for rec in reversed(tape):
        kind = rec[0]
        if kind == "rb":                        # t' = t + B(sp(A t)); cotangents gb, gdb of t'
            (nA, nB), x, xd, p, pd, a, ad = rec[1], rec[2], rec[3], rec[4], rec[5], rec[6], rec[7]
            dW[nB] += _wgrad3(a, gb) + _wgrad3(ad, gdb)
            ab, adb = nets.conv3x3_T(gb, W[nB]), nets.conv3x3_T(gdb, W[nB])
            s1 = _s1(p)
            pdb = s1 * adb
            pb = s1 * ab + s1 * (1 - s1) * pd * adb
            dW[nA] += _wgrad3(x, pb) + _wgrad3(xd, pdb)
            gb = gb + nets.conv3x3_T(pb, W[nA])
            gdb = gdb + nets.conv3x3_T(pdb, W[nA])
        elif kind == "up":                      # t = up(x) + s_l; cotangent of s_l = cotangent of t
            name, x, xd, l = rec[1], rec[2], rec[3], rec[4]
            skip_bar[l] = (gb, gdb)
            dW[name] += _wgrad_up(x, gb) + _wgrad_up(xd, gdb)
            gb, gdb = nets.up2x2_T(gb, W[name]), nets.up2x2_T(gdb, W[name])
        elif kind == "down":                    # x -> down(x) and x = s_l (skip)
            name, x, xd = rec[1], rec[2], rec[3]
            l = int(name[-1])
            dW[name] += _wgrad_down(x, gb) + _wgrad_down(xd, gdb)
            gb = nets.down2x2_T(gb, W[name]) + skip_bar[l][0]
            gdb = nets.down2x2_T(gdb, W[name]) + skip_bar[l][1]
        else:                                   # head: input cotangents not needed
            _, name, x, xd = rec
            dW[name] += _wgrad3(x, gb) + _wgrad3(xd, gdb)
    return dW


def flatten(net, dW):
    """dW dict -> fp64 vector in the weight-blob order (include/ideq.h)."""
    return np.concatenate([dW[k].ravel() for k in net.W.keys()])


def jfb_grads(net, fid, x_hat, x_star, lam, tau, step="grad"):
    """One image: loss, dL/dtheta (blob order), dL/dlam, dL/dtau, dL/dbeta (= 0)."""
    z = np.asarray(x_hat, dtype=np.float64)
    xs = np.asarray(x_star, dtype=np.float64)
    gg = net.grad_g(z)
    if step == "grad":
        gf = fid.grad(z)
        T = z - tau * (gf + lam * gg)
        r = T - xs
        v = r
        dlam = float(np.sum(r * (-tau * gg)))
        dtau = float(np.sum(r * (-(gf + lam * gg))))
    else:
        if fid.kind != "inpaint":
            raise NotImplementedError("JFB prox variant: inpainting (closed-form Jacobian) only")
        m, y = fid.m, fid.y
        vin = z - tau * lam * gg
        T = (tau * m * y + vin) / (tau * m + 1.0)
        r = T - xs
        v = r / (1.0 + tau * m)                                  # J_prox^T r (diagonal)
        dlam = float(np.sum(v * (-tau * gg)))
        dT_dtau = (m * y - lam * gg) / (1.0 + tau * m) - (tau * m * y + vin) * m / (1.0 + tau * m) ** 2
        dtau = float(np.sum(r * dT_dtau))
    loss = 0.5 * float(np.sum(r * r))
    dtheta = -tau * lam * flatten(net, phi_weight_grad(net, z, v))
    return loss, dtheta, dlam, dtau, 0.0
