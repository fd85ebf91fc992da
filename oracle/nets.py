"""Oracle networks N_theta and the gradient of g_theta (fp64, one image at a time).

g_theta(x) = 1/2 ||x - N_theta(x)||^2                      PAPER Eq. 2
grad g(x)  = (I - J_N(x))^T (x - N(x))                     Eq. 2 differentiated

Networks (BASELINE.json C1 and C2/C5; readings Q10, Q11, Q20 in DESIGN.md):
  tiny3 : N(x) = x + c3(sp(c2(sp(c1(x)))))                 BASELINE C1
  unet4 : head; per level 2 residual blocks t <- t + B(sp(A(t))); 2x2/s2 down;
          mirrored decoder with 2x2/s2 transposed up + additive skip; tail.
          N(x) = x + U(x)                                   BASELINE C2, C5
Convolutions are cross-correlations with zero padding (PyTorch convention).
The reverse pass is written out layer by layer (adjoint of each linear map,
softplus' = sigmoid); no autograd.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


# --------------------------------------------------------------------------- activations
def softplus(t):
    """sp(t) = log(1 + e^t), stable form max(t,0) + log1p(exp(-|t|)) (reading Q20)."""
    return np.maximum(t, 0.0) + np.log1p(np.exp(-np.abs(t)))


def softplus_grad(t):
    """sp'(t) = 1 / (1 + e^{-t}) (sigmoid)."""
    return 0.5 * (1.0 + np.tanh(0.5 * t))


def activation(t, act):
    return softplus(t) if act == "softplus" else t


def activation_grad(t, act):
    return softplus_grad(t) if act == "softplus" else np.ones_like(t)


# --------------------------------------------------------------------------- linear layers
def conv3x3(x, W):
    """out[co,m,n] = sum_{ci,a,b} W[co,ci,a,b] x[ci, m+a-1, n+b-1], zero outside
    (SURVEY §8(c)-4). x: [Cin][H][W], W: [Cout][Cin][3][3]."""
    Cin, H, Wd = x.shape
    xp = np.zeros((Cin, H + 2, Wd + 2))
    xp[:, 1:H + 1, 1:Wd + 1] = x
    out = np.zeros((W.shape[0], H * Wd))
    for a in range(3):
        for b in range(3):
            out += W[:, :, a, b] @ xp[:, a:a + H, b:b + Wd].reshape(Cin, H * Wd)
    return out.reshape(W.shape[0], H, Wd)


def conv3x3_T(g, W):
    """Adjoint of conv3x3 in its input: scatter each tap back,
    gin[ci, m+a-1, n+b-1] += sum_co W[co,ci,a,b] g[co,m,n]."""
    Cout, H, Wd = g.shape
    Cin = W.shape[1]
    gp = np.zeros((Cin, H + 2, Wd + 2))
    g2 = g.reshape(Cout, H * Wd)
    for a in range(3):
        for b in range(3):
            gp[:, a:a + H, b:b + Wd] += (W[:, :, a, b].T @ g2).reshape(Cin, H, Wd)
    return gp[:, 1:H + 1, 1:Wd + 1]


def down2x2(x, Wd):
    """out[co,i,j] = sum_{ci,a,b} Wd[co,ci,a,b] x[ci, 2i+a, 2j+b] (strided 2x2 conv)."""
    Cin, H, W = x.shape
    out = np.zeros((Wd.shape[0], (H // 2) * (W // 2)))
    for a in range(2):
        for b in range(2):
            out += Wd[:, :, a, b] @ x[:, a::2, b::2].reshape(Cin, -1)
    return out.reshape(Wd.shape[0], H // 2, W // 2)


def down2x2_T(g, Wd):
    """Adjoint of down2x2: gin[ci, 2i+a, 2j+b] = sum_co Wd[co,ci,a,b] g[co,i,j]."""
    Cout, h, w = g.shape
    Cin = Wd.shape[1]
    gin = np.zeros((Cin, 2 * h, 2 * w))
    g2 = g.reshape(Cout, -1)
    for a in range(2):
        for b in range(2):
            gin[:, a::2, b::2] = (Wd[:, :, a, b].T @ g2).reshape(Cin, h, w)
    return gin


def up2x2(x, Wu):
    """Transposed 2x2/s2 conv: out[co, 2i+a, 2j+b] = sum_ci Wu[ci,co,a,b] x[ci,i,j]."""
    Cin, h, w = x.shape
    Cout = Wu.shape[1]
    out = np.zeros((Cout, 2 * h, 2 * w))
    x2 = x.reshape(Cin, -1)
    for a in range(2):
        for b in range(2):
            out[:, a::2, b::2] = (Wu[:, :, a, b].T @ x2).reshape(Cout, h, w)
    return out


def up2x2_T(g, Wu):
    """Adjoint of up2x2: gin[ci,i,j] = sum_{co,a,b} Wu[ci,co,a,b] g[co, 2i+a, 2j+b]."""
    Cout, H, W = g.shape
    Cin = Wu.shape[0]
    gin = np.zeros((Cin, (H // 2) * (W // 2)))
    for a in range(2):
        for b in range(2):
            gin += Wu[:, :, a, b] @ g[:, a::2, b::2].reshape(Cout, -1)
    return gin.reshape(Cin, H // 2, W // 2)


# --------------------------------------------------------------------------- weight blob
def unpack_tiny(blob, C, w):
    """Blob order for tiny3 (include/ideq.h): conv1 [w][C][3][3], conv2 [w][w][3][3], conv3 [C][w][3][3]."""
    blob = np.asarray(blob, dtype=np.float64)
    shapes = [("c1", (w, C, 3, 3)), ("c2", (w, w, 3, 3)), ("c3", (C, w, 3, 3))]
    return _split(blob, shapes)


def unpack_unet(blob, C, widths, res_blocks=2):
    """Blob order for unet4 (include/ideq.h): head; for l=0..3 RB convs A,B per block
    then down_l (l<3); for l=2..0 up_l then RB convs; tail."""
    blob = np.asarray(blob, dtype=np.float64)
    w = list(widths)
    shapes = [("head", (w[0], C, 3, 3))]
    for l in range(4):
        for r in range(res_blocks):
            shapes += [(f"e{l}.{r}.A", (w[l], w[l], 3, 3)), (f"e{l}.{r}.B", (w[l], w[l], 3, 3))]
        if l < 3:
            shapes.append((f"down{l}", (w[l + 1], w[l], 2, 2)))
    for l in (2, 1, 0):
        shapes.append((f"up{l}", (w[l + 1], w[l], 2, 2)))
        for r in range(res_blocks):
            shapes += [(f"d{l}.{r}.A", (w[l], w[l], 3, 3)), (f"d{l}.{r}.B", (w[l], w[l], 3, 3))]
    shapes.append(("tail", (C, w[0], 3, 3)))
    return _split(blob, shapes)


def _split(blob, shapes):
    out, o = {}, 0
    for name, shp in shapes:
        n = int(np.prod(shp))
        out[name] = blob[o:o + n].reshape(shp)
        o += n
    if o != blob.size:
        raise ValueError(f"weight blob has {blob.size} values, layout needs {o}")
    return out


# --------------------------------------------------------------------------- networks
class Net:
    """N_theta for one architecture. ``U`` is the residual branch; N(x) = x + U(x)
    when identity_skip (BASELINE C1 "plus identity skip"), else N = U."""

    def __init__(self, arch, blob, C, widths, identity_skip=True, act="softplus", res_blocks=2):
        self.arch, self.C, self.act = arch, C, act
        self.identity_skip = bool(identity_skip)
        self.res_blocks = res_blocks
        if arch == "tiny3":
            self.W = unpack_tiny(blob, C, widths[0])
        elif arch == "unet4":
            self.W = unpack_unet(blob, C, widths, res_blocks)
        else:
            raise ValueError(arch)

    # ---- residual branch U and its input VJP
    def U_forward(self, x):
        """Returns U(x) and the saved pre-activations needed by the VJP."""
        if self.arch == "tiny3":
            return self._tiny_fwd(x)
        return self._unet_fwd(x)

    def U_vjp(self, saved, h):
        """J_U(x)^T h for the x that produced ``saved``."""
        if self.arch == "tiny3":
            return self._tiny_vjp(saved, h)
        return self._unet_vjp(saved, h)

    def _tiny_fwd(self, x):
        W, act = self.W, self.act
        p1 = conv3x3(x, W["c1"])
        p2 = conv3x3(activation(p1, act), W["c2"])
        u = conv3x3(activation(p2, act), W["c3"])
        return u, (p1, p2)

    def _tiny_vjp(self, saved, h):
        W, act = self.W, self.act
        p1, p2 = saved
        g = conv3x3_T(h, W["c3"]) * activation_grad(p2, act)
        g = conv3x3_T(g, W["c2"]) * activation_grad(p1, act)
        return conv3x3_T(g, W["c1"])

    def _unet_fwd(self, x):
        W, act, R = self.W, self.act, self.res_blocks
        saved = {}
        t = conv3x3(x, W["head"])
        skips = {}
        for l in range(4):
            for r in range(R):
                p = conv3x3(t, W[f"e{l}.{r}.A"])
                saved[f"e{l}.{r}"] = p
                t = t + conv3x3(activation(p, act), W[f"e{l}.{r}.B"])
            if l < 3:
                skips[l] = t
                t = down2x2(t, W[f"down{l}"])
        for l in (2, 1, 0):
            t = up2x2(t, W[f"up{l}"]) + skips[l]
            for r in range(R):
                p = conv3x3(t, W[f"d{l}.{r}.A"])
                saved[f"d{l}.{r}"] = p
                t = t + conv3x3(activation(p, act), W[f"d{l}.{r}.B"])
        u = conv3x3(t, W["tail"])
        return u, saved

    def _rb_vjp(self, g, p, WA, WB):
        """RB t' = t + B(sp(A t)):  dt = dt' + A^T( sp'(p) * B^T dt' )."""
        q = conv3x3_T(g, WB) * activation_grad(p, self.act)
        return g + conv3x3_T(q, WA)

    def _unet_vjp(self, saved, h):
        W, R = self.W, self.res_blocks
        g = conv3x3_T(h, W["tail"])
        skip_grad = {}
        for l in (0, 1, 2):
            for r in reversed(range(R)):
                g = self._rb_vjp(g, saved[f"d{l}.{r}"], W[f"d{l}.{r}.A"], W[f"d{l}.{r}.B"])
            skip_grad[l] = g                       # t = up(t_{l+1}) + s_l  =>  ds_l = dt
            g = up2x2_T(g, W[f"up{l}"])
        for l in (3, 2, 1, 0):
            if l < 3:
                g = down2x2_T(g, W[f"down{l}"]) + skip_grad[l]
            for r in reversed(range(R)):
                g = self._rb_vjp(g, saved[f"e{l}.{r}"], W[f"e{l}.{r}.A"], W[f"e{l}.{r}.B"])
        return conv3x3_T(g, W["head"])

    # ---- N, g and grad g
    def N(self, x):
        u, _ = self.U_forward(x)
        return x + u if self.identity_skip else u

    def g(self, x):
        """g(x) = 1/2 ||x - N(x)||^2 (Eq. 2)."""
        e = x - self.N(x)
        return 0.5 * float(np.sum(e * e))

    def grad_g(self, x):
        """grad g(x) = (I - J_N)^T (x - N(x)) with J_N^T e = [skip] e + J_U^T e (Eq. 2)."""
        u, saved = self.U_forward(x)
        n = x + u if self.identity_skip else u
        e = x - n
        jnt_e = self.U_vjp(saved, e) + (e if self.identity_skip else 0.0)
        return e - jnt_e
