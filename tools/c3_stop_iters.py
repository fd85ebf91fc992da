"""Print the per-image stop iterations of the CUDA path's full-size C3 early-stopping solve
(bf16, tol 1e-4): used to pick long-running sample images for tools/make_golden_c3_stop.py."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_19705_b200 import configs, ideq, synth  # noqa: E402

cfg = configs.get("C3")
prob = synth.make_problem(cfg)
s = ideq.Solver(cfg, prob["weights"], precision="bf16", max_batch=cfg["batch"])
s.set_operator(prob)
x = torch.tensor(prob["x0"]).cuda()
st, _, _ = s.solve(torch.tensor(prob["y"]).cuda(), x, s.params(tol=1e-4))
print(json.dumps({"iters": st["iters"].tolist(), "status": st["status"].tolist(),
                  "residual": [float(r) for r in st["residual"]]}))
