"""Thin ctypes binding of the C ABI in ``include/ideq.h`` (argument marshalling only).

Every step of the iteration runs inside ``lib/libideq.so`` (hand-written sm_100a
kernels). There is no Python or CPU fallback: if the library is missing or no
B200 is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IDEQ_LIB") or os.path.join(_HERE, "lib", "libideq.so")  # IDEQ_LIB: A/B builds

# ---- enums (include/ideq.h)
OK, E_INVALID, E_DIVERGED, E_UNSUPPORTED, E_CUDA, E_NCCL, E_NOMEM, E_STATE = range(8)
STATUS_NAMES = ["OK", "INVALID", "DIVERGED", "UNSUPPORTED", "CUDA", "NCCL", "NOMEM", "STATE"]
PREC = {"fp32": 0, "bf16": 1}
ARCH = {"tiny3": 0, "unet4": 1}
ACT = {"softplus": 0, "identity": 1}
OP = {"blur": 0, "inpaint": 1, "phase": 2, "rician": 3, "mri": 4}
STEP = {"grad": 0, "prox": 1}
BLUR = {"direct": 0, "fft": 1}
STOP = {"per_image": 0, "global_max": 1}
KCLASS = ["conv_tc", "conv_simt", "headtail", "fidelity", "step", "reduce"]


class NetDesc(C.Structure):
    _fields_ = [("arch", C.c_int), ("channels", C.c_int), ("widths", C.c_int * 4), ("res_blocks", C.c_int),
                ("identity_skip", C.c_int), ("act", C.c_int), ("weights", C.POINTER(C.c_float)),
                ("n_weights", C.c_size_t)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("nccl_id", C.c_ubyte * 128)]


class OperatorDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("step", C.c_int), ("blur_impl", C.c_int), ("ksize", C.c_int),
                ("kernel_per_image", C.c_int), ("kernels", C.POINTER(C.c_float)),
                ("masks", C.POINTER(C.c_ubyte)), ("n_phase", C.c_int), ("phase_masks", C.POINTER(C.c_float)),
                ("sigma", C.c_float)]


class Params(C.Structure):
    _fields_ = [("lam", C.c_float), ("tau", C.c_float), ("beta", C.c_float), ("max_iter", C.c_int),
                ("tol", C.c_float), ("check_every", C.c_int), ("stop_rule", C.c_int), ("restart", C.c_int),
                ("restart_B", C.c_float), ("averaging", C.c_int), ("compute_frozen", C.c_int)]


class PlanOpts(C.Structure):
    _fields_ = [("micro_batch", C.c_int), ("workspace_bytes", C.c_size_t)]


class ImageStat(C.Structure):
    _fields_ = [("iters", C.c_int), ("residual", C.c_float), ("status", C.c_int), ("restarts", C.c_int),
                ("k0", C.c_int)]


class Profile(C.Structure):
    _fields_ = [("ms", C.c_double * 6), ("launches", C.c_longlong * 6), ("flops", C.c_double * 6),
                ("bytes", C.c_double * 6)]


SYMBOLS = ["ideq_get_nccl_id", "ideq_create", "ideq_set_operator", "ideq_solve", "ideq_solve_host", "ideq_grad_g",
           "ideq_fidelity_grad", "ideq_fidelity_prox", "ideq_set_profiling", "ideq_get_profile",
           "ideq_launches_per_iteration", "ideq_last_error", "ideq_destroy", "ideq_abi_version", "ideq_debug_conv",
           "ideq_jfb_grad", "ideq_create_ex", "ideq_get_plan", "ideq_time_class", "ideq_debug_rb",
           "ideq_debug_set_fusion"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libideq.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing; build it with `python -m paper_2605_19705_b200.build`")
    lib = C.CDLL(path)
    vp, i, f, fp = C.c_void_p, C.c_int, C.c_float, C.POINTER(C.c_float)
    lib.ideq_get_nccl_id.argtypes = [C.POINTER(C.c_ubyte)]
    lib.ideq_create.argtypes = [C.POINTER(NetDesc), i, i, vp, i, i, i, C.POINTER(Dist), C.POINTER(vp)]
    lib.ideq_create_ex.argtypes = [C.POINTER(NetDesc), i, i, vp, i, i, i, C.POINTER(Dist), C.POINTER(PlanOpts),
                                   C.POINTER(vp)]
    lib.ideq_get_plan.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_size_t)]
    lib.ideq_time_class.argtypes = [vp, i, i, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
    lib.ideq_set_operator.argtypes = [vp, C.POINTER(OperatorDesc), i]
    lib.ideq_solve.argtypes = [vp, vp, vp, i, C.POINTER(Params), C.POINTER(ImageStat), fp]
    lib.ideq_solve_host.argtypes = [vp, vp, vp, i, C.POINTER(Params), C.POINTER(ImageStat), fp]
    lib.ideq_grad_g.argtypes = [vp, vp, vp, vp, i]
    lib.ideq_fidelity_grad.argtypes = [vp, vp, vp, vp, i]
    lib.ideq_fidelity_prox.argtypes = [vp, vp, vp, f, vp, i]
    lib.ideq_set_profiling.argtypes = [vp, i]
    lib.ideq_get_profile.argtypes = [vp, C.POINTER(Profile), i]
    lib.ideq_launches_per_iteration.argtypes = [vp]
    lib.ideq_launches_per_iteration.restype = i
    lib.ideq_last_error.argtypes = [vp]
    lib.ideq_last_error.restype = C.c_char_p
    lib.ideq_destroy.argtypes = [vp]
    lib.ideq_destroy.restype = None
    lib.ideq_abi_version.restype = i
    for s in SYMBOLS:
        if s not in ("ideq_last_error", "ideq_destroy", "ideq_abi_version", "ideq_launches_per_iteration"):
            getattr(lib, s).restype = i
    _lib = lib
    return lib


class IdeqError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"ideq {STATUS_NAMES[code] if 0 <= code < 8 else code}: {msg}")
        self.code = code


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _ptr(t):
    """Device pointer of a torch tensor (or an int address)."""
    if t is None:
        return None
    if isinstance(t, int):
        return C.c_void_p(t)
    return C.c_void_p(t.data_ptr())


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = (C.c_ubyte * 128)()
    r = lib.ideq_get_nccl_id(buf)
    if r != OK:
        raise IdeqError(r, "ncclGetUniqueId failed")
    return bytes(buf)


class Solver:
    """One ideq_ctx: a network, an operator and solver workspaces on one device."""

    def __init__(self, cfg: dict, weights: np.ndarray, precision: str = None, device: int = 0, stream=None,
                 max_batch: int = None, H: int = None, W: int = None, rank: int = 0, world: int = 1,
                 nccl_id: bytes = None, micro_batch: int = 0, workspace_bytes: int = 0):
        self.lib = load_library()
        self.cfg = cfg
        self.C = cfg["C"]
        self.H = cfg["H"] if H is None else H
        self.W = cfg["W"] if W is None else W
        self.max_batch = cfg["batch"] if max_batch is None else max_batch
        prec = cfg["precision"] if precision is None else precision
        self.precision = prec
        self._w = np.ascontiguousarray(weights, dtype=np.float32)
        nd = NetDesc()
        nd.arch = ARCH[cfg["net"]]
        nd.channels = cfg["C"]
        for k, w in enumerate(cfg["widths"]):
            nd.widths[k] = int(w)
        nd.res_blocks = cfg.get("res_blocks", 2)
        nd.identity_skip = int(cfg.get("identity_skip", True))
        nd.act = ACT[cfg.get("act", "softplus")]
        nd.weights = _fptr(self._w)
        nd.n_weights = self._w.size
        dist = None
        if nccl_id is not None:  # NCCL communicator (also for world == 1: single-rank all-reduce)
            dist = Dist()
            dist.rank, dist.world = rank, world
            C.memmove(dist.nccl_id, nccl_id, 128)
        ctx = C.c_void_p()
        s = None if stream is None else C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
        opts = PlanOpts(int(micro_batch), int(workspace_bytes))
        r = self.lib.ideq_create_ex(C.byref(nd), PREC[prec], device, s, self.max_batch, self.H, self.W,
                                    C.byref(dist) if dist is not None else None, C.byref(opts), C.byref(ctx))
        self.ctx = ctx
        if r != OK:
            msg = self.lib.ideq_last_error(ctx).decode() if ctx.value else "invalid create arguments"
            self.close()
            raise IdeqError(r, msg)

    # ---------------------------------------------------------------- helpers
    def _check(self, r, allow=(OK,)):
        if r not in allow:
            raise IdeqError(r, self.lib.ideq_last_error(self.ctx).decode())
        return r

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            self.lib.ideq_destroy(self.ctx)
        self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- operator
    def set_operator(self, prob: dict, batch: int = None, step: str = None, blur_impl: str = None):
        cfg = self.cfg
        op = OperatorDesc()
        op.kind = OP[cfg["op"]]
        op.step = STEP[cfg["step"] if step is None else step]
        op.blur_impl = BLUR[(cfg.get("blur_impl", "direct") if blur_impl is None else blur_impl)]
        self._keep = []
        if cfg["op"] == "blur":
            if cfg.get("kernel_per_image", False):
                k = np.ascontiguousarray(prob["kernels"], dtype=np.float32)
                op.kernel_per_image = 1
            else:
                k = np.ascontiguousarray(prob["kernel"], dtype=np.float32)[None]
                op.kernel_per_image = 0
            op.ksize = k.shape[-1]
            op.kernels = _fptr(k)
            self._keep.append(k)
        elif cfg["op"] == "inpaint":
            m = np.ascontiguousarray(prob["masks"], dtype=np.uint8)
            op.masks = m.ctypes.data_as(C.POINTER(C.c_ubyte))
            self._keep.append(m)
        elif cfg["op"] == "rician":
            op.sigma = float(cfg["sigma"])
        elif cfg["op"] == "mri":
            m = np.ascontiguousarray(prob["kmask"], dtype=np.uint8)
            op.masks = m.ctypes.data_as(C.POINTER(C.c_ubyte))
            self._keep.append(m)
        else:
            d = np.ascontiguousarray(prob["phase_masks"], dtype=np.float32)
            op.n_phase = d.shape[0]
            op.phase_masks = _fptr(d)
            self._keep.append(d)
        nb = len(prob["images"]) if batch is None else batch
        self._check(self.lib.ideq_set_operator(self.ctx, C.byref(op), nb))

    # ---------------------------------------------------------------- solve
    def params(self, lam=None, tau=None, beta=None, max_iter=None, tol=None, check_every=None, stop_rule=None,
               restart=0, restart_B=0.0, averaging=False, compute_frozen=False):
        cfg = self.cfg
        p = Params()
        p.lam = cfg["lam"] if lam is None else lam
        p.tau = cfg["tau"] if tau is None else tau
        p.beta = cfg["beta"] if beta is None else beta
        p.max_iter = cfg["max_iter"] if max_iter is None else max_iter
        p.tol = cfg["tol"] if tol is None else tol
        p.check_every = cfg["check_every"] if check_every is None else check_every
        p.stop_rule = STOP[cfg["stop_rule"] if stop_rule is None else stop_rule]
        p.restart = int(restart)
        p.restart_B = float(restart_B)
        p.averaging = int(bool(averaging))
        p.compute_frozen = int(bool(compute_frozen))
        return p

    def solve(self, y, x, params: Params, trace: bool = False, batch: int = None):
        """Device solve: y, x are CUDA tensors (x updated in place). Returns (stats, status, trace)."""
        n = x.shape[0] if batch is None else batch
        stats = (ImageStat * n)()
        tr = np.full(params.max_iter, np.nan, dtype=np.float32) if trace else None
        r = self.lib.ideq_solve(self.ctx, _ptr(y), _ptr(x), n, C.byref(params), stats,
                                _fptr(tr) if trace else None)
        self._check(r, allow=(OK, E_DIVERGED))
        return _stats(stats), r, tr

    def solve_host(self, y: np.ndarray, x: np.ndarray, params: Params, trace: bool = False):
        """Host solve: y, x are C-contiguous float32 numpy arrays (x updated in place)."""
        assert y.dtype == np.float32 and x.dtype == np.float32 and y.flags.c_contiguous and x.flags.c_contiguous
        n = x.shape[0]
        stats = (ImageStat * n)()
        tr = np.full(params.max_iter, np.nan, dtype=np.float32) if trace else None
        r = self.lib.ideq_solve_host(self.ctx, C.c_void_p(y.ctypes.data), C.c_void_p(x.ctypes.data), n,
                                     C.byref(params), stats, _fptr(tr) if trace else None)
        self._check(r, allow=(OK, E_DIVERGED))
        return _stats(stats), r, tr

    # ---------------------------------------------------------------- components
    def grad_g(self, z, out, u_out=None):
        self._check(self.lib.ideq_grad_g(self.ctx, _ptr(z), _ptr(out), _ptr(u_out), z.shape[0]))

    def fidelity_grad(self, y, x, out):
        self._check(self.lib.ideq_fidelity_grad(self.ctx, _ptr(y), _ptr(x), _ptr(out), x.shape[0]))

    def fidelity_prox(self, y, v, tau, out):
        self._check(self.lib.ideq_fidelity_prox(self.ctx, _ptr(y), _ptr(v), float(tau), _ptr(out), v.shape[0]))

    def jfb_grad(self, y, x_hat, x_star, params):
        """JFB gradient at x_hat (include/ideq.h ideq_jfb_grad): (loss, dtheta[n_weights], dlam, dtau, dbeta)."""
        dth = np.zeros(self._w.size, dtype=np.float32)
        out = [C.c_float() for _ in range(4)]
        self._check(self.lib.ideq_jfb_grad(self.ctx, _ptr(y), _ptr(x_hat), _ptr(x_star), x_hat.shape[0],
                                           C.byref(params), dth.ctypes.data_as(C.c_void_p),
                                           *[C.byref(o) for o in out]))
        dlam, dtau, dbeta, loss = (o.value for o in out)
        return loss, dth, dlam, dtau, dbeta

    # ---------------------------------------------------------------- profiling
    def set_profiling(self, on: bool):
        self._check(self.lib.ideq_set_profiling(self.ctx, int(on)))

    def profile(self, reset: bool = True) -> dict:
        p = Profile()
        self._check(self.lib.ideq_get_profile(self.ctx, C.byref(p), int(reset)))
        return {k: dict(ms=p.ms[i], launches=p.launches[i], flops=p.flops[i], bytes=p.bytes[i])
                for i, k in enumerate(KCLASS)}

    def plan(self) -> dict:
        """The workspace plan chosen at create (ideq_get_plan)."""
        mb, nb = C.c_int(), C.c_size_t()
        self._check(self.lib.ideq_get_plan(self.ctx, C.byref(mb), C.byref(nb)))
        return {"micro_batch": mb.value, "workspace_bytes": nb.value}

    def time_class(self, cls: str, reps: int = 10) -> dict:
        """In-graph timing of one kernel class of the last solve's iteration (ideq_time_class):
        ms per iteration and the class's algorithmic FLOPs / bytes per iteration."""
        ms, fl, by, it = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        self._check(self.lib.ideq_time_class(self.ctx, KCLASS.index(cls), int(reps), C.byref(ms), C.byref(fl),
                                             C.byref(by), C.byref(it)))
        return {"ms": ms.value, "flops": fl.value, "bytes": by.value, "iter_ms": it.value,
                "share": ms.value / it.value if it.value > 0 else None}

    def set_fusion(self, on: bool):
        """include/ideq_debug.h ideq_debug_set_fusion: fused level-0 residual blocks on / off."""
        fn = self.lib.ideq_debug_set_fusion
        fn.argtypes = [C.c_void_p, C.c_int]
        fn.restype = C.c_int
        self._check(fn(self.ctx, int(on)))

    def launches_per_iteration(self) -> int:
        return int(self.lib.ideq_launches_per_iteration(self.ctx))


def debug_conv(kind: int, precision: str, use_tc: bool, w: np.ndarray, N: int, Hin: int, Win: int, inp, out,
               aux=None, epi: int = 0):
    """include/ideq_debug.h: run one network conv layer on device NHWC tensors."""
    lib = load_library()
    fn = lib.ideq_debug_conv
    fn.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_char_p, C.c_int]
    fn.restype = C.c_int
    w = np.ascontiguousarray(w, dtype=np.float32)
    err = C.create_string_buffer(256)
    r = fn(kind, PREC[precision], int(use_tc), _fptr(w), w.shape[0], w.shape[1], N, Hin, Win, _ptr(inp), _ptr(out),
           _ptr(aux), epi, err, 256)
    if r != OK:
        raise IdeqError(r, err.value.decode())


def debug_rb(vjp: bool, wA: np.ndarray, wB: np.ndarray, N: int, H: int, W: int, x, out, act):
    """include/ideq_debug.h: one fused level-0 residual block on device NHWC bf16 tensors."""
    lib = load_library()
    fn = lib.ideq_debug_rb
    fn.argtypes = [C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int, C.c_int, C.c_int, C.c_void_p,
                   C.c_void_p, C.c_void_p, C.c_char_p, C.c_int]
    fn.restype = C.c_int
    wa = np.ascontiguousarray(wA, dtype=np.float32)
    wb = np.ascontiguousarray(wB, dtype=np.float32)
    err = C.create_string_buffer(256)
    r = fn(int(vjp), _fptr(wa), _fptr(wb), N, H, W, _ptr(x), _ptr(out), _ptr(act), err, 256)
    if r != OK:
        raise IdeqError(r, err.value.decode())


def _stats(stats):
    return dict(iters=np.array([s.iters for s in stats]), residual=np.array([s.residual for s in stats]),
                status=np.array([s.status for s in stats]), restarts=np.array([s.restarts for s in stats]),
                k0=np.array([s.k0 for s in stats]))
