"""A/B of the fused level-0 residual block (rbf.cu) against the unfused conv_tc pair on C3:
time per iteration (graph-captured solve, tol=0) and the max difference of the iterates."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_19705_b200 import configs, ideq, synth
cfg = configs.get(os.environ.get("CFG", "C3"))
prob = synth.make_problem(cfg)
y = torch.tensor(prob["y"]).cuda(); x0 = torch.tensor(prob["x0"]).cuda()
K = int(os.environ.get("ITERS", "50"))
outs = {}
for on in (0, 1, 0, 1):
    s = ideq.Solver(cfg, prob["weights"], precision="bf16")
    s.set_operator(prob); s.set_fusion(bool(on))
    p = s.params(max_iter=K, tol=0.0)
    x = x0.clone(); s.solve(y, x, p); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x = x0.clone(); e0.record(); s.solve(y, x, p); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    outs[on] = x
    print(f"fused={on} {ms / K * 1000:.1f} us/iter  {cfg['batch'] * K / ms * 1000:.0f} img-it/s")
print("max|fused-unfused| =", (outs[1] - outs[0]).abs().max().item())
