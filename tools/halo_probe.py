"""Probe the UMMA descriptor encoding of row-shifted halo windows on the GPU (one conv layer)."""
import os, subprocess, sys
code = r'''
import numpy as np, sys
sys.path.insert(0, ".")
from oracle import nets
from tests.gpu_util import bf16_round, from_nhwc_dev, nhwc_dev, rel_l2
import torch
from paper_2605_19705_b200 import ideq
for (ci, co) in [(32, 32), (64, 64)]:
    rng = np.random.default_rng(0)
    w = (rng.standard_normal((co, ci, 3, 3)) / np.sqrt(ci * 9)).astype(np.float32)
    x = rng.standard_normal((2, ci, 4, 272))
    ref = np.stack([nets.conv3x3(bf16_round(x)[n], bf16_round(w)) for n in range(2)])
    out = torch.zeros((2, 4, 272, co), device="cuda", dtype=torch.bfloat16)
    ideq.debug_conv(0, "bf16", True, w, 2, 4, 272, nhwc_dev(x, "bf16"), out, None, 0)
    print("mode", sys.argv[1], (ci, co), "rel", rel_l2(from_nhwc_dev(out), ref))
'''
for m in ["3", "0"]:
    env = dict(os.environ, IDEQ_NO_HALO=("1" if m == "3" else "0"))
    r = subprocess.run([sys.executable, "-c", code, m], env=env, capture_output=True, text=True, timeout=120)
    print(r.stdout.strip(), r.stderr.strip()[-300:])
