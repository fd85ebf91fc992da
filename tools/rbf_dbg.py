import numpy as np, torch, sys, os, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) == 1:
    for dbg in (7487 | 8192, 63, 0):
        try:
            r = subprocess.run([sys.executable, __file__, str(dbg)], capture_output=True, text=True, timeout=40)
            print("dbg", dbg, "rc", r.returncode, (r.stdout + r.stderr).strip().splitlines()[-1:])
        except subprocess.TimeoutExpired:
            print("dbg", dbg, "TIMEOUT")
    sys.exit(0)
from paper_2605_19705_b200 import ideq
dbg = int(sys.argv[1])
N, H, W = 1, 3, 128
rng = np.random.default_rng(0)
wA = (rng.standard_normal((32, 32, 3, 3)) * 0.05).astype(np.float32)
x = torch.randn(N, H, W, 32, device="cuda").to(torch.bfloat16)
out = torch.zeros_like(x); act = torch.zeros_like(x)
ideq.debug_rb(dbg << 8, wA, wA, N, H, W, x, out, act)
print("ok", out.float().abs().mean().item())
