"""One eager (profiled-mode) C3 iteration for ncu captures: every kernel of one step, once."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_19705_b200 import configs, ideq, synth
name = os.environ.get("CFG", "C3")
cfg = configs.get(name, **({"batch": int(os.environ["BATCH"])} if "BATCH" in os.environ else {}))
prob = synth.make_problem(cfg)
s = ideq.Solver(cfg, prob["weights"], precision=cfg.get("precision", "bf16"))
s.set_operator(prob)
if "FUSE" in os.environ: s.set_fusion(os.environ["FUSE"] == "1")
y = torch.tensor(prob["y"]).cuda(); x = torch.tensor(prob["x0"]).cuda()
s.set_profiling(True)
s.solve(y, x, s.params(max_iter=int(os.environ.get("ITERS", "1")), tol=0.0))
prof = s.profile()
print({k: round(v["ms"], 3) for k, v in prof.items()})
