"""Error map of the fused residual block (forward) against the oracle for a few shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import nets
from tests.gpu_util import bf16_round, from_nhwc_dev, nhwc_dev, torch_cuda
from paper_2605_19705_b200 import ideq
torch = torch_cuda()
for (W, H, N) in [(128, 300, 1), (128, 1, 300), (128, 5, 70), (256, 300, 1)]:
    rng = np.random.default_rng(1)
    wA = (rng.standard_normal((32, 32, 3, 3)) * np.sqrt(2.0 / 288)).astype(np.float32)
    wB = (rng.standard_normal((32, 32, 3, 3)) * np.sqrt(2.0 / 288)).astype(np.float32)
    x = rng.standard_normal((N, 32, H, W))
    xr, ar, br = bf16_round(x), bf16_round(wA), bf16_round(wB)
    a_ref = np.stack([nets.softplus(nets.conv3x3(xr[n], ar)) for n in range(N)])
    out_ref = np.stack([xr[n] + nets.conv3x3(bf16_round(a_ref)[n], br) for n in range(N)])
    xd = nhwc_dev(x, "bf16"); out = torch.zeros_like(xd); act = torch.zeros_like(xd)
    ideq.debug_rb(False, wA, wB, N, H, W, xd, out, act)
    for name, got, ref in (("act", from_nhwc_dev(act), a_ref), ("out", from_nhwc_dev(out), out_ref)):
        err = np.abs(got - ref) > 2.0 ** -7 * np.abs(ref).max()
        print(W, H, N, name, "bad", int(err.sum()), "of", err.size)
        if err.any():
            nh = np.argwhere(err.any(axis=(1, 3)))  # (n, h)
            print("   bad (n,h):", nh[:12].tolist(), "count", len(nh))
            ws = np.argwhere(err.any(axis=(0, 1, 2)))
            print("   bad w:", ws[:20].ravel().tolist(), "count", len(ws))
            cs = np.argwhere(err.any(axis=(0, 2, 3)))
            print("   bad c:", cs.ravel().tolist()[:40])
