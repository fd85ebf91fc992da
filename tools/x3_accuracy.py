"""Accuracy of one network convolution in the fp32 mode's two arithmetic forms against the fp64
oracle layer: FFMA (fp32 CUDA cores) and 3xTF32 (tcgen05 kind::tf32, 3 MMAs per product), for
growing contraction depth K = 9 x C_in. Prints relative L2 and max |err| / max |ref|."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import nets  # noqa: E402
from paper_2605_19705_b200 import ideq  # noqa: E402

rng = np.random.default_rng(0)
for c in (32, 64, 128, 256, 512):
    N, H, W = 2, 16, 24
    w = (rng.standard_normal((c, c, 3, 3)) * np.sqrt(2.0 / (9 * c)) * 0.3).astype(np.float32)
    x = rng.uniform(0.0, 1.0, (N, c, H, W)).astype(np.float32)   # softplus outputs are >= 0
    ref = np.stack([nets.conv3x3(x[n].astype(np.float64), w.astype(np.float64)) for n in range(N)])
    xin = torch.tensor(np.ascontiguousarray(x.transpose(0, 2, 3, 1))).cuda()
    for tc in (False, True):
        out = torch.zeros((N, H, W, c), device="cuda", dtype=torch.float32)
        ideq.debug_conv(0, "fp32", tc, w, N, H, W, xin, out, None, 0)
        got = out.cpu().numpy().transpose(0, 3, 1, 2).astype(np.float64)
        err = got - ref
        print(f"C={c:4d} K={9 * c:5d} {'3xTF32' if tc else 'FFMA  '}: rel_l2 {np.linalg.norm(err) / np.linalg.norm(ref):.2e}"
              f"  max|err|/max|ref| {np.abs(err).max() / np.abs(ref).max():.2e}  mean err/rms {err.mean() / np.sqrt((ref ** 2).mean()):+.1e}",
              flush=True)
