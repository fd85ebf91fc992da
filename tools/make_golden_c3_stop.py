"""Write tests/golden/c3_stop_oracle.npz: the fp64 ORACLE's early-stopping iteration of BASELINE
config C3 at full size (3 x 256 x 256, U-Net-32, inpainting prox, beta 0.7, per-image stop at
tol 1e-4, max_iter 300; PAPER P:796 / P:860, Alg. 2) for sampled images of the 32-image batch.
Per image: the residual after every update up to 10 updates past the oracle's stop (or the cap),
the stop iteration and status, and the iterate at the stop. Calls only oracle/ and the seeded
input generator; tests/test_gpu_livelist.py compares the CUDA path's live-image-list solve
against it.

    python tools/make_golden_c3_stop.py [image ...]     # default: 0 31 (~2 s per image-iteration)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import solver as osolver  # noqa: E402
from paper_2605_19705_b200 import configs, synth  # noqa: E402

TOL = 1e-4
MARGIN = 10


def main(images):
    cfg = configs.get("C3")
    K = cfg["max_iter"]
    out = {}
    for i in images:
        t0 = time.time()
        sub = synth.make_problem(cfg, images=[i])
        net = osolver.make_net(cfg, sub["weights"])
        fid = osolver.make_fidelities(cfg, sub)[0]
        x = sub["x0"][0].astype(np.float64)
        xp = x.copy()
        trace, k_stop, x_stop = [], None, None
        for k in range(K):
            xn = osolver.ideq_step(x, xp, net, fid, cfg["lam"], cfg["tau"], cfg["beta"], cfg["step"])
            r = osolver.residual(xn, x)
            trace.append(r)
            xp, x = x, xn
            if k_stop is None and r <= TOL:
                k_stop, x_stop = k + 1, x.copy()
            if k_stop is not None and k + 1 >= k_stop + MARGIN:
                break
        if k_stop is None:
            k_stop, x_stop = K, x.copy()
        out[f"iters_{i}"] = np.int64(k_stop)
        out[f"status_{i}"] = np.int64(0 if trace[k_stop - 1] <= TOL else 1)
        out[f"rtrace_{i}"] = np.array(trace)
        out[f"x_{i}"] = x_stop.astype(np.float32)
        print(f"image {i}: stop {k_stop} r {trace[k_stop - 1]:.4e} ({time.time() - t0:.0f} s)", flush=True)
    out["images"] = np.array(images)
    out["tol"] = np.float64(TOL)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c3_stop_oracle.npz"), **out)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [0, 31])
